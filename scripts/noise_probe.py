"""Real noise budget (bits) left in the deepest intermediates of the hot path,
per limb count: decode score/value accumulators and prefill diagonals / P.V."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2602_08798_b200 as cg  # noqa: E402
from paper_2602_08798_b200.arcc import broadcast_wave  # noqa: E402
from paper_2602_08798_b200.backend import GpuContext  # noqa: E402
from paper_2602_08798_b200.linear_kernels import fold_wave  # noqa: E402

L = int(os.environ.get("CGB_LIMBS", "4"))
params = cg.BackendParams()
n, p, d2 = params.n_slots, params.plain_modulus, 64
ctx = GpuContext(params, 0, n_limbs=L)
C = GpuContext
fp = cg.FixedPointParams(8, p)
rng = np.random.default_rng(0)
tok = lambda r, c: np.mod(np.round(rng.uniform(-1, 1, (r, c)) * 256).astype(np.int64), p)
K = cg.encode(tok(128, d2), cg.EncodingKind.OUTER, ctx)
V = cg.encode(tok(128, d2), cg.EncodingKind.OUTER, ctx)
q = ctx.encrypt(ctx.plain_from_dense(tok(1, d2)[0]))
out = {"L": L, "q_bits": ctx._ring.q_bits, "fresh": ctx.noise_budget_bits(q)}
# decode scores: 64 broadcasts (one-hot, 14 rotations) x mult_cipher, summed
qw = C.wave_of([q] * d2, [ctx] * d2)
b = broadcast_wave(qw, np.arange(d2), n)
out["broadcast"] = ctx.noise_budget_bits(b.handles()[5])
prods = C.w_mult_cipher(b, C.wave_of(K.parts, [ctx] * d2))
acc = C.w_sum(prods, [np.arange(d2)]).handles()[0]
out["decode_scores"] = ctx.noise_budget_bits(acc)
# decode values: fresh weights x V_c, full fold, one-hot mask, summed
a = ctx.encrypt(ctx.plain_from_dense(tok(1, 128)[0]))
pv = C.w_mult_cipher(C.wave_of([a] * d2, [ctx] * d2), C.wave_of(V.parts, [ctx] * d2))
tot = fold_wave(pv, n)
from paper_2602_08798_b200.backend import onehot_batch  # noqa: E402
pieces = C.w_mult_plain(tot, onehot_batch(n, np.arange(d2)))
o = C.w_sum(pieces, [np.arange(d2)]).handles()[0]
out["decode_values"] = ctx.noise_budget_bits(o)
# prefill diagonal r: K column tiled to period 128, rotated, times Q column, summed over 64 columns
kt = cg.encodings.tile_wave(C.wave_of(K.parts, [ctx] * d2), 128, n // 128)
kr = C.w_rotate(kt, 77)
Q = cg.encode(tok(128, d2), cg.EncodingKind.OUTER, ctx)
dg = C.w_sum(C.w_mult_cipher(C.wave_of(Q.parts, [ctx] * d2), kr), [np.arange(d2)]).handles()[0]
out["prefill_diag"] = ctx.noise_budget_bits(dg)
# prefill P.V column: 128 weight rows x V_c, fold, one-hot, summed
rows = C.w_encrypt([ctx] * 128, np.stack([ctx.plain_from_dense(tok(1, 128)[0]) for _ in range(128)]))
pr = C.w_mult_cipher(rows, C.wave_of([V.parts[0]] * 128, [ctx] * 128))
pc = C.w_sum(C.w_mult_plain(fold_wave(pr, n), onehot_batch(n, np.arange(128))), [np.arange(128)]).handles()[0]
out["prefill_pv"] = ctx.noise_budget_bits(pc)
print(json.dumps(out))
