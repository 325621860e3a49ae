"""Hot-path scenarios, written once against the reference's public API.

``api`` is any namespace exposing the reference names (BackendParams,
FixedPointParams, fp_encode, encode, EncodingKind, pack_token_inner,
init_cache, append_token, maybe_refresh, attention_step,
prefill_attention, MpcChannel, fold_sum, broadcast_slot, tile_token,
arcc_inner_inner, arcc_inner_outer, compact_scores, cpvm_inner_diagonal,
cpmm_outer_diagonal, decode).  ``new_ctx(params, seed)`` builds the
context.  make_golden.py runs these against the reference
(/root/reference/pkg/src/cryptogen) to record tests/golden/*.npz; the
tests run them against this repo's host code over the slot oracle (CPU),
the polynomial oracle (CPU) and the B200 backend (GPU).
"""

from __future__ import annotations

import json

import numpy as np

ID_BASE = 1_000_000_000


def _tokens(api, rng, fp, p, rows, d):
    return np.mod(api.fp_encode(rng.uniform(-1.0, 1.0, (rows, d)), fp), p)


def _record(ctx, snap, mpc=None, extra=None):
    rec = {"delta": json.dumps(ctx.counter.delta(snap), sort_keys=True)}
    if mpc is not None:
        rec["transcript"] = json.dumps(mpc.transcript)
        rec["mpc_bytes"] = np.int64(mpc.bytes_sent)
        rec["mpc_rounds"] = np.int64(mpc.rounds)
        rec["next_mask"] = mpc.sample_mask(4)
    if extra:
        rec.update(extra)
    return rec


def build_cache(api, ctx, fp, rng, m, t, d2):
    p = ctx.params.plain_modulus
    if m:
        K = api.encode(_tokens(api, rng, fp, p, m, d2), api.EncodingKind.OUTER, ctx)
        V = api.encode(_tokens(api, rng, fp, p, m, d2), api.EncodingKind.OUTER, ctx)
        cache = api.init_cache(K, V, ctx)
    else:
        cache = api.init_cache(None, None, ctx, d2=d2)
    for _ in range(t):
        k = api.pack_token_inner(_tokens(api, rng, fp, p, 1, d2)[0], ctx)
        v = api.pack_token_inner(_tokens(api, rng, fp, p, 1, d2)[0], ctx)
        cache = api.append_token(cache, k, v, ctx)
    return cache


def attention(api, new_ctx, n, p, d2, m, t, seed=0, f=8, refresh=False):
    params = api.BackendParams(n_slots=n, plain_modulus=p)
    ctx = new_ctx(params, seed)
    fp = api.FixedPointParams(f, p)
    rng = np.random.default_rng(seed)
    cache = build_cache(api, ctx, fp, rng, m, t, d2)
    mpc = api.MpcChannel(p, seed=seed + 11)
    if refresh:
        cache = api.maybe_refresh(cache, ctx, mpc, force=True)
    q = api.pack_token_inner(_tokens(api, rng, fp, p, 1, d2)[0], ctx)
    snap = ctx.counter.snapshot()
    out = api.attention_step(q, cache, fp, ctx, mpc)
    rec = _record(ctx, snap, mpc)
    rec["out"] = ctx.decrypt(out)[:d2].astype(np.int64)
    rec["out_budget"] = np.int64(out.noise_budget)
    rec["out_id"] = np.int64(out.id % ID_BASE)
    return rec, (ctx, out)


def attention_heads(api, new_ctx, n, p, d2, m, t, heads, seed=0, f=8):
    """H heads, forked contexts and per-head channels, run sequentially."""
    params = api.BackendParams(n_slots=n, plain_modulus=p)
    root = new_ctx(params, seed)
    fp = api.FixedPointParams(f, p)
    rng = np.random.default_rng(seed)
    ctxs, caches, qs, chans = [], [], [], []
    for h in range(heads):
        c = root.fork()
        ctxs.append(c)
        caches.append(build_cache(api, c, fp, rng, m, t, d2))
        qs.append(api.pack_token_inner(_tokens(api, rng, fp, p, 1, d2)[0], c))
        chans.append(api.MpcChannel(p, seed=seed + 100 + h))
    return root, fp, ctxs, caches, qs, chans


def prefill(api, new_ctx, n, p, d2, m, seed=0, f=8):
    params = api.BackendParams(n_slots=n, plain_modulus=p)
    ctx = new_ctx(params, seed)
    fp = api.FixedPointParams(f, p)
    rng = np.random.default_rng(seed)
    Q, K, V = (api.encode(_tokens(api, rng, fp, p, m, d2), api.EncodingKind.OUTER, ctx) for _ in range(3))
    mpc = api.MpcChannel(p, seed=seed + 7)
    snap = ctx.counter.snapshot()
    O = api.prefill_attention(Q, K, V, fp, ctx, mpc, causal=True)
    rec = _record(ctx, snap, mpc)
    rec["out"] = api.decode(O, ctx).astype(np.int64)
    rec["out_budgets"] = np.array([pt.noise_budget for pt in O.parts], np.int64)
    return rec, (ctx, O)


def cache_ops(api, new_ctx, n, p, d2, steps, seed=0, f=8):
    """Appends interleaved with forced refreshes; returns decoded segments."""
    params = api.BackendParams(n_slots=n, plain_modulus=p)
    ctx = new_ctx(params, seed)
    fp = api.FixedPointParams(f, p)
    rng = np.random.default_rng(seed)
    cache = build_cache(api, ctx, fp, rng, 3, 0, d2)
    mpc = api.MpcChannel(p, seed=seed + 3)
    snap = ctx.counter.snapshot()
    for s in range(steps):
        k = api.pack_token_inner(_tokens(api, rng, fp, p, 1, d2)[0], ctx)
        v = api.pack_token_inner(_tokens(api, rng, fp, p, 1, d2)[0], ctx)
        cache = api.append_token(cache, k, v, ctx)
        if s % 3 == 2:
            cache = api.maybe_refresh(cache, ctx, mpc, force=True)
    rec = _record(ctx, snap, mpc)
    rec["auto_K"] = api.decode(cache.auto_K, ctx).astype(np.int64)
    rec["auto_V"] = api.decode(cache.auto_V, ctx).astype(np.int64)
    rec["budgets"] = np.array([pt.noise_budget for _, seg in cache.segments() for pt in seg.parts], np.int64)
    rec["refresh_log"] = json.dumps([[e.step, e.segment, e.part_index, e.part_id % ID_BASE, e.budget_before,
                                      e.mpc_bytes, e.forced] for e in cache.refresh_log])
    return rec, (ctx, cache)


def kernels(api, new_ctx, n, p, seed=0):
    """Small known-answer runs of every L1/L2 kernel on the hot path."""
    params = api.BackendParams(n_slots=n, plain_modulus=p)
    ctx = new_ctx(params, seed)
    rng = np.random.default_rng(seed)
    rec = {}
    snap = ctx.counter.snapshot()
    a = ctx.encrypt(rng.integers(0, p, n))
    rec["fold_8"] = ctx.decrypt(api.fold_sum(a, 8, ctx))
    rec["fold_n"] = ctx.decrypt(api.fold_sum(a, n, ctx))
    rec["bcast"] = ctx.decrypt(api.broadcast_slot(a, 5, n, ctx))
    rec["bcast_w"] = ctx.decrypt(api.broadcast_slot(a, 3, 6, ctx))
    x = ctx.encrypt(ctx.plain_from_dense(rng.integers(0, p, 4)))
    rec["tile"] = ctx.decrypt(api.tile_token(x, 4, 5, ctx))
    d = 4
    Kc = api.encode(rng.integers(0, 50, (6, d)), api.EncodingKind.OUTER, ctx)
    q = ctx.encrypt(ctx.plain_from_dense(rng.integers(0, 50, d)))
    rec["ii_outer"] = ctx.decrypt(api.arcc_inner_inner(q, Kc, ctx).ct)
    Ki = api.encode(rng.integers(0, 50, (d, 5)), api.EncodingKind.INNER, ctx)
    rec["ii_inner"] = ctx.decrypt(api.arcc_inner_inner(q, Ki, ctx).ct)
    B = n // d
    Kq = api.encode(rng.integers(0, 50, (B + 3, d)), api.EncodingKind.INNER_COMPACTED, ctx)
    qq = ctx.encrypt(ctx.plain_from_dense(rng.integers(0, 50, B + 3)))
    rec["ii_comp"] = ctx.decrypt(api.arcc_inner_inner(qq, Kq, ctx).ct)
    sv = api.arcc_inner_outer(q, Kq, ctx)
    rec["io_comp"] = np.stack([ctx.decrypt(pt) for pt in sv.parts])
    rec["compact"] = ctx.decrypt(api.compact_scores(sv, ctx).ct)
    Kn = api.encode(rng.integers(0, 50, (7, d)), api.EncodingKind.INNER, ctx)
    sv2 = api.arcc_inner_outer(q, Kn, ctx)
    rec["io_inner"] = np.stack([ctx.decrypt(pt) for pt in sv2.parts])
    W = api.encode(rng.integers(-20, 20, (6, 3)), api.EncodingKind.DIAGONAL, ctx, encrypted=False)
    xv = ctx.encrypt(ctx.plain_from_dense(rng.integers(0, 30, 6)))
    rec["cpvm"] = ctx.decrypt(api.cpvm_inner_diagonal(xv, W, ctx))
    X = api.encode(rng.integers(0, 30, (5, 6)), api.EncodingKind.OUTER, ctx)
    rec["cpmm"] = api.decode(api.cpmm_outer_diagonal(X, W, ctx), ctx)
    rec["delta"] = json.dumps(ctx.counter.delta(snap), sort_keys=True)
    return {k: (np.asarray(v, np.int64) if not isinstance(v, str) else v) for k, v in rec.items()}, ctx


def op_program(api, new_ctx, n, p, steps=200, seed=0):
    """The reference's random op program (tests/test_backend.py:169-197 shape)."""
    ctx = new_ctx(api.BackendParams(n_slots=n, plain_modulus=p), 1)
    rng = np.random.default_rng(seed)
    ct = ctx.encrypt(rng.integers(0, p, n))
    other = rng.integers(0, p, n)
    oct_ = ctx.encrypt(other)
    for _ in range(steps):
        op = rng.integers(0, 5)
        if op == 0:
            ct = ctx.add(ct, oct_)
        elif op == 1:
            ct = ctx.add_plain(ct, rng.integers(0, p, n))
        elif op == 2:
            ct = ctx.mult_plain(ct, rng.integers(0, p, n))
        elif op == 3:
            ct = ctx.mult_cipher(ct, oct_)
        else:
            ct = ctx.rotate(ct, int(rng.integers(0, n)))
        ct = ctx.with_budget(ct, 190)
    return {"out": ctx.decrypt(ct).astype(np.int64), "counter": json.dumps(ctx.counter.as_dict(), sort_keys=True)}, ctx


# scenario table: name -> (function, kwargs) ; P64 = default_plain_modulus(64, 26)
P64 = 67109633
P8192 = 536903681
SMALL = {
    "attn_m5_t0": (attention, dict(n=64, p=P64, d2=4, m=5, t=0)),
    "attn_m0_t19": (attention, dict(n=64, p=P64, d2=4, m=0, t=19)),
    "attn_m5_t19": (attention, dict(n=64, p=P64, d2=4, m=5, t=19)),
    "attn_m16_t40_refresh": (attention, dict(n=64, p=P64, d2=4, m=16, t=40, refresh=True)),
    "prefill_m5": (prefill, dict(n=64, p=P64, d2=4, m=5)),
    "prefill_m8": (prefill, dict(n=64, p=P64, d2=4, m=8)),
    "cache_ops": (cache_ops, dict(n=64, p=P64, d2=4, steps=20)),
    "kernels": (kernels, dict(n=64, p=P64)),
    "op_program": (op_program, dict(n=64, p=P64)),
}
FULL = {
    "full_attn_m128": (attention, dict(n=8192, p=P8192, d2=64, m=128, t=0)),
    "full_attn_m96_t32": (attention, dict(n=8192, p=P8192, d2=64, m=96, t=32)),
    "full_attn_m0_t130": (attention, dict(n=8192, p=P8192, d2=64, m=0, t=130)),
    "full_prefill_m128": (prefill, dict(n=8192, p=P8192, d2=64, m=128)),
}
