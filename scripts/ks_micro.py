"""Batched key-switch microbenchmark on one ring: COUNT ciphertexts rotated by one
step (one key, like a doubling step of the decode broadcast chains) or by distinct
steps.  Prints one JSON line: us per key switch (CUDA events over REPS calls), the
per-kernel table of one call, and -- under ncu with --nvtx-include "ks/" -- exactly
one batched key switch is captured (the NVTX range 'ks')."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_08798_b200 import _native  # noqa: E402
from paper_2602_08798_b200.ring import Ring  # noqa: E402

LOGN = int(os.environ.get("KS_LOGN", "14"))
L = int(os.environ.get("KS_L", "3"))
COUNT = int(os.environ.get("KS_COUNT", "768"))
REPS = int(os.environ.get("KS_REPS", "10"))
MODE = os.environ.get("KS_MODE", "rotate_add")  # rotate | rotate_add | distinct
T = {13: 536903681, 14: 536903681, 15: 537133057, 16: 537133057}[LOGN]
_native.build()
g = Ring(LOGN, T, L, 1 << (LOGN - 1), True, np.arange(8, dtype=np.uint32) * 7 + 1, arena_cts=2 * COUNT + 8,
         arena_pts=4, q_bits=49)
g.set_stream(torch.cuda.current_stream().cuda_stream)
src = g.alloc(COUNT)
rng = np.random.default_rng(0)
g.encrypt(rng.integers(0, T, (COUNT, g.n_slots)), np.arange(8, dtype=np.uint32) + 1000, 0, src)
steps = (np.arange(1, COUNT + 1) if MODE == "distinct" else np.full(COUNT, 64)).astype(np.int64)
out = g.alloc(COUNT)
add = MODE == "rotate_add"
for _ in range(2):
    g.rotate(src, steps, out, add_input=add)
torch.cuda.synchronize()
if os.environ.get("KS_PROFILE"):
    torch.cuda.nvtx.range_push("ks")
    g.rotate(src, steps, out, add_input=add)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    sys.exit(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(REPS):
    g.rotate(src, steps, out, add_input=add)
e1.record()
torch.cuda.synchronize()
us = 1e3 * e0.elapsed_time(e1) / (REPS * COUNT)
g.timing(1)
g.rotate(src, steps, out, add_input=add)
rep = g.timing_report()
g.timing(0)
kern = {k: {"launches": v[0], "ms": round(v[1], 4), "GBps": round(v[2] / (v[1] * 1e6), 1) if v[1] > 0 else None,
            "Gmodmul_s": round(v[3] / (v[1] * 1e6), 1) if v[1] > 0 and v[3] else None}
        for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1]) if not k.startswith("(")}
ctw = 2 * L * (1 << LOGN) * 8
alg = 2 * ctw + (8 * 2 * L * (L + 1) * (1 << LOGN)) / (1 if MODE != "distinct" else 1) / COUNT
print(json.dumps({"logN": LOGN, "L": L, "count": COUNT, "mode": MODE, "us_per_keyswitch": us,
                  "algorithmic_bytes_per_item": alg, "kernels": kern}))
