"""Hoisted vs per-item key switch on the production ring (logN 14, L = 3, 49-bit
primes): K rotations of ONE ciphertext by K distinct steps (the CPVM's diagonal
steps -> hoisted path) against K distinct ciphertexts rotated by the same K
steps (per-item path).  Prints per-rotation device time and the kernel table."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_08798_b200 import _native  # noqa: E402
from paper_2602_08798_b200.ring import Ring  # noqa: E402

K = int(os.environ.get("HOIST_K", "256"))
_native.build()
g = Ring(14, 536903681, 3, 8192, True, np.arange(8, dtype=np.uint32) * 7 + 1, arena_cts=2 * K + 8, arena_pts=4,
         q_bits=49)
g.set_stream(torch.cuda.current_stream().cuda_stream)
rng = np.random.default_rng(0)
src = g.alloc(K)
for i in range(K):
    g.encrypt(rng.integers(0, 536903681, 8192), np.arange(8, dtype=np.uint32) + 1000, i, src[i:i + 1])
steps = np.arange(1, K + 1, dtype=np.int64)
out = g.alloc(K)
res = {}
for mode, a in (("hoisted", np.repeat(src[:1], K)), ("per_item", src)):
    for _ in range(2):  # keys built, warm
        g.rotate(a, steps, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.rotate(a, steps, out)
    e1.record()
    torch.cuda.synchronize()
    g.timing(True)
    g.rotate(a, steps, out)
    torch.cuda.synchronize()
    rep = g.timing_report()
    g.timing(False)
    res[mode] = {"us_per_rotation": 1e3 * e0.elapsed_time(e1) / (5 * K),
                 "kernels": {k: {"launches": v[0], "ms": round(v[1], 4),
                                 "GBps": round(v[2] / (v[1] * 1e6), 1) if v[1] > 0 else None}
                             for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1]) if not k.startswith("(")}}
print(json.dumps({"K": K, "ring": "logN14 L3 q49 P49", **res}))
