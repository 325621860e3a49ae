"""cProfile of one decode step (host side) on the GPU box."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_08798_b200 as api  # noqa: E402
from paper_2602_08798_b200.backend import GpuContext  # noqa: E402

root, fp, ctxs, caches, chans, rng = bench.build_state(api, GpuContext, 128, 12)
C = GpuContext
toks = [C.w_encrypt([c for c in ctxs for _ in range(3)], np.stack(bench.step_tokens(rng, 12))).handles()
        for _ in range(3)]


def step(t):
    cs = api.maybe_refresh_heads(caches, ctxs, chans)
    cs = api.append_token_heads(cs, t[1::3], t[2::3], ctxs)
    return api.attention_step_heads(t[0::3], cs, fp, ctxs, chans)


step(toks[0])
torch.cuda.synchronize()
t0 = time.perf_counter()
step(toks[1])
torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t0) * 1e3)
pr = cProfile.Profile()
pr.enable()
step(toks[2])
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
