"""Sequential per-op restatement of the reference decode hot path.

TEST / BASELINE INFRASTRUCTURE ONLY.  Executes the reference's op sequence
one ``ctx`` call at a time, exactly as /root/reference/pkg/src/cryptogen
does it:

  broadcast_slot          arcc.py:80-94
  arcc_inner_inner OUTER  arcc.py:113-121
  arcc_inner_outer COMP.  arcc.py:170-176 (tile_token encodings.py:196-216,
                          fold_sum linear_kernels.py:27-42)
  _dot_into_slot          arcc.py:222-231
  attention_step          arcc.py:320-379
  prefill_attention       arcc.py:248-317 (_column_period :234-245)
  _append_one/append      kv_cache.py:114-143
  _refresh_part/refresh   kv_cache.py:146-196
  he_to_shares etc.       nonlinear.py:101-144

Two uses: (1) over the slot oracle (``oracle.slots.SlotContext``) it is the
reference's CPU path -- bench.py times it as ``--impl reference`` and as
the ``cpu_baseline`` leg; (2) over ``GpuContext`` it is the per-op drop-in
path, which tests/test_gpu_hotpath.py compares word-for-word with the
fused wave schedule.  Cache and score containers are the host package's
data classes (plain dataclasses, no computation).
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np

from paper_2602_08798_b200.encodings import EncodingKind, PackedMatrix
from paper_2602_08798_b200.fixedpoint import attention_weights, fp_truncate, from_signed, to_signed
from paper_2602_08798_b200.kv_cache import RefreshEvent
from paper_2602_08798_b200.nonlinear import SharePair


def _one_hot(n, j):
    v = np.zeros(n, dtype=np.int64)
    v[j] = 1
    return v


def fold_sum(a, block, ctx):
    out, step = a, 1
    while step < block:
        out = ctx.add(out, ctx.rotate(out, step))
        step *= 2
    return out


def tile_token(x, d, B, ctx):
    out, copies = x, 1
    while copies < B:
        out = ctx.add(out, ctx.rotate(out, -(copies * d)))
        copies *= 2
    return out


def broadcast_slot(a, j, width, ctx):
    out = ctx.rotate(ctx.mult_plain(a, _one_hot(ctx.params.n_slots, j)), j)
    filled = 1
    while filled < width:
        out = ctx.add(out, ctx.rotate(out, -filled))
        filled *= 2
    return out


def reconstruct(s):
    return to_signed((s.client + s.server) % s.p, s.p)


def share_vector(values, ch):
    secret = from_signed(values, ch.p)
    r = ch.sample_mask(secret.shape[0])
    return SharePair((secret - r) % ch.p, r, ch.p, secret.shape[0])


def he_to_shares(ct, ctx, ch, length=None):
    n, p = ctx.params.n_slots, ctx.params.plain_modulus
    length = n if length is None else length
    r = ch.sample_mask(n)
    client = ctx.decrypt(ctx.add_plain(ct, (p - r) % p))
    ch.transfer("he_to_shares", n)
    return SharePair(client[:length].copy(), r[:length].copy(), p, length)


def shares_to_he(s, ctx, ch):
    out = ctx.add_plain(ctx.encrypt(ctx.plain_from_dense(s.client)), ctx.plain_from_dense(s.server))
    ch.transfer("shares_to_he", ctx.params.n_slots)
    return out


def truncate(s, fp, ch):
    out = fp_truncate(reconstruct(s), fp.f)
    ch.transfer("truncate", s.length, trips=3)
    return share_vector(out, ch)


def attention_step(q, cache, fp, ctx, mpc):
    m, t, d2, B = cache.m, cache.t_auto, cache.d2, cache.B
    n = ctx.params.n_slots
    pieces = []
    if m > 0:
        acc = None
        for j, part in enumerate(cache.prefill_K.parts):
            prod = ctx.mult_cipher(broadcast_slot(q, j, n, ctx), part)
            acc = prod if acc is None else ctx.add(acc, prod)
        pieces.append(reconstruct(he_to_shares(acc, ctx, mpc, length=m)))
    if t > 0:
        vt = tile_token(q, d2, B, ctx)
        for qi, part in enumerate(cache.auto_K.parts):
            sc = fold_sum(ctx.mult_cipher(vt, part), d2, ctx)
            vals = reconstruct(he_to_shares(sc, ctx, mpc))
            pieces.append(vals[np.arange(min(B, t - qi * B)) * d2])
    a = attention_weights(np.concatenate(pieces), d2, fp)
    mpc.transfer("decode_softmax", m + t, trips=3 + fp.reciprocal_iters)
    o = None
    if m > 0:
        a_pref = shares_to_he(share_vector(a[:m], mpc), ctx, mpc)
        for c in range(d2):
            prod = ctx.mult_cipher(a_pref, cache.prefill_V.parts[c])
            piece = ctx.mult_plain(fold_sum(prod, n, ctx), _one_hot(n, c))
            o = piece if o is None else ctx.add(o, piece)
    if t > 0:
        acc = None
        for qi, part in enumerate(cache.auto_V.parts):
            rows = min(B, t - qi * B)
            coeff = np.zeros(n, dtype=np.int64)
            coeff[: rows * d2] = np.repeat(a[m + qi * B: m + qi * B + rows], d2)
            prod = ctx.mult_cipher(shares_to_he(share_vector(coeff, mpc), ctx, mpc), part)
            acc = prod if acc is None else ctx.add(acc, prod)
        step = d2
        while step < n:
            acc = ctx.add(acc, ctx.rotate(acc, step))
            step *= 2
        o = acc if o is None else ctx.add(o, acc)
    return shares_to_he(truncate(he_to_shares(o, ctx, mpc, length=d2), fp, mpc), ctx, mpc)


def _append_one(seg, token, pos, mask, ctx, fresh):
    new = ctx.mult_plain(ctx.rotate(token, -pos) if pos else token, mask)
    parts = list(seg.parts)
    if fresh:
        parts.append(ctx.add(ctx.encrypt(ctx.zeros()), new))
    else:
        parts[-1] = ctx.add(parts[-1], new)
    return PackedMatrix(replace(seg.encoding, rows=seg.encoding.rows + 1), parts, encrypted=True)


def append_token(cache, k, v, ctx):
    b = cache.t_auto % cache.B
    pos = b * cache.d2
    mask = np.zeros(ctx.params.n_slots, dtype=np.int64)
    mask[pos: pos + cache.d2] = 1
    return replace(cache, t_auto=cache.t_auto + 1, auto_K=_append_one(cache.auto_K, k, pos, mask, ctx, b == 0),
                   auto_V=_append_one(cache.auto_V, v, pos, mask, ctx, b == 0))


def maybe_refresh(cache, ctx, ch, force=False):
    params = ctx.params
    n, p, thr = params.n_slots, params.plain_modulus, params.refresh_threshold
    new, events = {}, []
    for name, seg in cache.segments():
        parts, changed = list(seg.parts), False
        for i, part in enumerate(parts):
            if force or part.noise_budget <= thr:
                events.append(RefreshEvent(cache.t_auto, name, i, part.id, part.noise_budget,
                                           2 * params.ciphertext_bytes(), force and part.noise_budget > thr))
                r = ch.sample_mask(n)
                fresh = ctx.encrypt(ctx.decrypt(ctx.add_plain(part, (p - r) % p)))
                ch.transfer("refresh", n, trips=2)
                parts[i] = ctx.add_plain(fresh, r)
                ctx.counter.refresh_events += 1
                changed = True
        if changed:
            new[name] = PackedMatrix(seg.encoding, parts, encrypted=True, slot_period=seg.slot_period)
    if not new:
        return cache
    return replace(cache, prefill_K=new.get("prefill_K", cache.prefill_K),
                   prefill_V=new.get("prefill_V", cache.prefill_V), auto_K=new.get("auto_K", cache.auto_K),
                   auto_V=new.get("auto_V", cache.auto_V), refresh_log=cache.refresh_log + tuple(events))


def _column_period(P, idx, period, ctx):
    col = P.parts[idx]
    if P.slot_period == period:
        return col
    return tile_token(col, period, ctx.params.n_slots // period, ctx)


def prefill_attention(Q, K, V, fp, ctx, mpc, causal=True):
    """arcc.py:248-317 op by op (score diagonals from rotated key columns,
    client softmax, value sweep by _dot_into_slot arcc.py:222-231)."""
    from paper_2602_08798_b200.encodings import next_pow2
    from paper_2602_08798_b200.fixedpoint import attention_weights, causal_attention_weights

    m, d2 = Q.encoding.rows, Q.encoding.cols
    n = ctx.params.n_slots
    w = next_pow2(m)
    k_cols = [_column_period(K, c, w, ctx) for c in range(d2)]
    diag_shares = []
    for r in range(w):
        acc = None
        for c in range(d2):
            kr = ctx.rotate(k_cols[c], r) if r else k_cols[c]
            prod = ctx.mult_cipher(Q.parts[c], kr)
            acc = prod if acc is None else ctx.add(acc, prod)
        diag_shares.append(he_to_shares(acc, ctx, mpc, length=m))
    S = np.zeros((m, m), dtype=np.int64)
    for r, sp in enumerate(diag_shares):
        vals = reconstruct(sp)
        for i in range(m):
            j = (i + r) % w
            if j < m:
                S[i, j] = vals[i]
    A = np.stack([causal_attention_weights(S[i], i, d2, fp) if causal else attention_weights(S[i], d2, fp)
                  for i in range(m)])
    mpc.transfer("prefill_softmax", m * m, trips=3 + fp.reciprocal_iters)
    a_rows = [shares_to_he(share_vector(A[i], mpc), ctx, mpc) for i in range(m)]
    out_parts = []
    for c in range(d2):
        acc = None
        for i in range(m):
            prod = ctx.mult_cipher(a_rows[i], V.parts[c])
            piece = ctx.mult_plain(fold_sum(prod, n, ctx), _one_hot(n, i))
            acc = piece if acc is None else ctx.add(acc, piece)
        sp = truncate(he_to_shares(acc, ctx, mpc, length=m), fp, mpc)
        out_parts.append(shares_to_he(sp, ctx, mpc))
    return PackedMatrix(Q.encoding, out_parts, encrypted=True, slot_period=None)
