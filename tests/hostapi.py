"""This repo's host modules as one namespace (same names as the reference)."""
from types import SimpleNamespace


def repo_api():
    from paper_2602_08798_b200 import arcc, backend, encodings, fixedpoint, kv_cache, linear_kernels, nonlinear

    ns = SimpleNamespace()
    for mod in (backend, encodings, fixedpoint, kv_cache, linear_kernels, nonlinear, arcc):
        for k in dir(mod):
            if not k.startswith("__"):
                setattr(ns, k, getattr(mod, k))
    return ns


def compare(rec, gold, keys=None):
    """Assert a scenario record equals the golden record (all shared keys)."""
    import numpy as np

    keys = keys or [k for k in gold.files]
    for k in keys:
        g = gold[k]
        r = rec[k]
        if g.dtype.kind in "US":
            assert str(r) == str(g), f"{k}: {r} != {g}"
        else:
            assert np.array_equal(np.asarray(r), g), f"{k} differs:\n{np.asarray(r)}\nvs golden\n{g}"
