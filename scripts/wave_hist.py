"""Batch sizes of the key-switch / mult_cipher calls of one decode step (12 heads, L = 128),
and the per-item cost of a batched key switch as a function of the batch size."""
import collections
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_08798_b200 as api  # noqa: E402
from paper_2602_08798_b200.backend import GpuContext  # noqa: E402
from paper_2602_08798_b200.ring import Ring  # noqa: E402

calls = []
for name in ("rotate", "galois", "mult_cipher", "mult_cipher_ext", "mult_cipher_ext2", "rotate_hoisted"):
    if hasattr(Ring, name):
        def wrap(fn, name=name):
            def w(self, a, *args, **kw):
                calls.append((name, len(a)))
                return fn(self, a, *args, **kw)
            return w
        setattr(Ring, name, wrap(getattr(Ring, name)))

root, fp, ctxs, caches, chans, rng = bench.build_state(api, GpuContext, 128, 12)
C = GpuContext
toks = [C.w_encrypt([c for c in ctxs for _ in range(3)], np.stack(bench.step_tokens(rng, 12))).handles() for _ in range(3)]
for i in range(3):
    calls.clear()
    cs = api.maybe_refresh_heads(caches, ctxs, chans)
    cs = api.append_token_heads(cs, toks[i][1::3], toks[i][2::3], ctxs)
    api.attention_step_heads(toks[i][0::3], cs, fp, ctxs, chans)
    caches = cs
torch.cuda.synchronize()
hist = collections.Counter(calls)
print(json.dumps({"calls": sorted(([k[0], k[1], v] for k, v in hist.items()), key=lambda r: (r[0], -r[1]))}))
ring = ctxs[0].ring
T = ring.t
for count in (12, 24, 48, 96, 192, 384, 768):
    src = ring.alloc(count); out = ring.alloc(count)
    ring.encrypt(np.zeros((count, ring.n_slots), dtype=np.int64), np.arange(8, dtype=np.uint32) + 5, 0, src)
    steps = np.full(count, 64, dtype=np.int64)
    for _ in range(3):
        ring.rotate(src, steps, out, add_input=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(4, 1536 // count)
    e0.record()
    for _ in range(reps):
        ring.rotate(src, steps, out, add_input=True)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"count": count, "us_per_call": 1e3 * e0.elapsed_time(e1) / reps, "us_per_item": 1e3 * e0.elapsed_time(e1) / reps / count}))
    ring.free(src); ring.free(out)
