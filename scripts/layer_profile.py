"""cProfile of config-3 decode steps (host side) on the GPU box: the caches are
built by encode (config 4's shortcut), then `steps` decode steps of the layer."""
import cProfile
import os
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("CGB_PT_ARENA_GIB", "12")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_08798_b200 as api  # noqa: E402
from paper_2602_08798_b200.backend import BackendParams, GpuContext  # noqa: E402

args = bench.parse()
M, mdl = bench.layer_model(args)
ctx = GpuContext(BackendParams(), 0)
rng = np.random.default_rng(0)
caches = [[api.init_cache(*(api.encode(bench.fp_tokens(rng, args.L, 64), api.EncodingKind.OUTER, ctx)
                            for _ in range(2)), ctx) for _ in range(12)]]
state = M.GenerationState(position=args.L, caches=caches, next_logits=np.zeros(8, np.int64))
chans = M.channels(0, 1, 12, bench.P)
_, state = M.decode_step(mdl, state, ctx, chans, force_refresh=True)  # warm (weights, keys)
torch.cuda.synchronize()
for refresh in (True, False):
    t0 = time.perf_counter()
    _, state = M.decode_step(mdl, state, ctx, chans, force_refresh=refresh)
    torch.cuda.synchronize()
    print(f"decode step (force_refresh={refresh}): {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
_, state = M.decode_step(mdl, state, ctx, chans, force_refresh=True)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(40)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

if os.environ.get("LAYER_PROF_PREFILL"):
    prompt = np.random.default_rng(0).integers(0, bench.GPT2_VOCAB, args.L).tolist()
    chans = M.channels(0, 1, 12, bench.P)
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    M.prefill(mdl, prompt, ctx, chans)
    torch.cuda.synchronize()
    pr.disable()
    print(f"prefill: {time.perf_counter() - t0:.2f} s", flush=True)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
