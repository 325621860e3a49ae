"""Record golden vectors of the hot-path scenarios from the REFERENCE itself.

Run here (the reference is importable only in this container):
    python tests/golden/make_golden.py [--full]
It imports cryptogen from /root/reference/pkg/src, runs every scenario of
harness.py against the reference's own Context (slot emulation) and
writes tests/golden/<name>.npz.  The committed .npz files are what the
tests compare against; /root/reference is never read at test time.
"""
import sys
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))

import harness  # noqa: E402


def reference_api():
    from cryptogen import arcc, backend, encodings, fixedpoint, kv_cache, linear_kernels, nonlinear

    ns = SimpleNamespace()
    for mod in (backend, encodings, fixedpoint, kv_cache, linear_kernels, nonlinear, arcc):
        for k in dir(mod):
            if not k.startswith("__"):
                setattr(ns, k, getattr(mod, k))
    return ns, backend.new_context


def main():
    api, new_ctx = reference_api()
    table = dict(harness.SMALL)
    if "--full" in sys.argv:
        table.update(harness.FULL)
    for name, (fn, kw) in table.items():
        t0 = time.time()
        rec, _ = fn(api, new_ctx, **kw)
        np.savez_compressed(HERE / f"{name}.npz", **rec)
        print(f"{name}: {time.time() - t0:.2f}s", flush=True)


if __name__ == "__main__":
    main()
