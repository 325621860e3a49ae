"""Host profile + GPU time of the 12-head prefill attention (config 2)."""
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

root = GpuContext(api.BackendParams(), 0)
fp = api.FixedPointParams(bench.F, bench.P)
rng = np.random.default_rng(0)
ctxs = [root.fork() for _ in range(12)]
mats = [[api.encode(bench.fp_tokens(rng, 128, 64), api.EncodingKind.OUTER, c) for _ in range(3)] for c in ctxs]
chans = [api.MpcChannel(bench.P, seed=2000 + h) for h in range(12)]
run = lambda: api.prefill_attention_heads([m[0] for m in mats], [m[1] for m in mats], [m[2] for m in mats], fp, ctxs,
                                          chans)
run()
torch.cuda.synchronize()
ring = root.ring
ring.timing(True)
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
run()
torch.cuda.synchronize()
pr.disable()
print(f"prefill wall {time.perf_counter() - t0:.2f} s")
rep = ring.timing_report()
ring.timing(False)
ks = sorted(((k, v) for k, v in rep.items() if not k.startswith("(")), key=lambda kv: -kv[1][1])
print("kernel ms total", sum(v[1] for _, v in ks), "idle", rep.get("(idle)"))
for k, v in ks[:10]:
    print(f"  {k:20s} {v[0]:6d} {v[1]:9.1f} ms")
for k, v in rep.items():
    if k.startswith("(trans:"):
        print("  ", k, v[0], round(v[1], 1))
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
