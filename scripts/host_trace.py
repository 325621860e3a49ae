"""Host timeline of decode steps (CGB_HOST_TRACE): ms between the phase marks of
arcc.attention_step_heads, plus the GPU time of the same step (CUDA events)."""
import os
import sys
import time
from pathlib import Path

os.environ["CGB_HOST_TRACE"] = "1"
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_08798_b200 as api  # noqa: E402
from paper_2602_08798_b200 import arcc  # noqa: E402
from paper_2602_08798_b200.backend import GpuContext  # noqa: E402

root, fp, ctxs, caches, chans, rng = bench.build_state(api, GpuContext, 128, 12)
C = GpuContext
toks = [C.w_encrypt([c for c in ctxs for _ in range(3)], np.stack(bench.step_tokens(rng, 12))).handles()
        for _ in range(5)]


def step(t):
    cs = api.maybe_refresh_heads(caches, ctxs, chans)
    cs = api.append_token_heads(cs, t[1::3], t[2::3], ctxs)
    return api.attention_step_heads(t[0::3], cs, fp, ctxs, chans)


for i in range(5):
    torch.cuda.synchronize()
    arcc._TRACE.clear()
    t0 = time.perf_counter()
    step(toks[i])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if i >= 2:
        marks = [("call", t0)] + arcc._TRACE + [("synced", t1)]
        print(" | ".join(f"{b[0]} +{(b[1] - a[1]) * 1e3:.2f}" for a, b in zip(marks, marks[1:])),
              f"|| wall {(t1 - t0) * 1e3:.2f} ms")
