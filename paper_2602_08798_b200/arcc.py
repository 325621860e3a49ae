"""Cipher-cipher attention over the heterogeneous encrypted KV cache.

Mirrors /root/reference/pkg/src/cryptogen/arcc.py: ``broadcast_slot``
(:80-94), ``arcc_inner_inner`` (:97-152), ``arcc_inner_outer`` (:155-195),
``compact_scores`` (:198-214), ``_dot_into_slot`` (:222-231),
``_column_period`` (:234-245), ``prefill_attention`` (:248-317) and
``attention_step`` (:320-379), with the same signatures.

B200 design: the reference evaluates one op at a time; here every set of
independent chains becomes one *wave* (a batch of ciphertexts processed by
one launch sequence).  A decode step of H heads is a fixed schedule:

  scores   1 x mult_plain(one-hot)   H*d2 items
           1 x rotate(j)             H*d2 items (per-item Galois element)
           13 x rotate_add(-2^s)     H*d2 items (shared key -> streamed once)
           1 x mult_cipher + sum     H*d2 -> H
           tile 7 + mult_cipher + fold 6 over the generated segment
  client   masked decrypt, softmax, re-encrypt       (H channels)
  values   1 x mult_cipher           H*d2 items
           13 x rotate_add(2^s)      H*d2 items
           1 x mult_plain(one-hot) + sum, generated segment fold 7
  client   masked decrypt, truncate, re-encrypt

All ops are exact functions of their inputs (integer arithmetic mod q), so
the batched schedule yields the same ciphertext words as the per-op
reference sequence; counters, ledger budgets, ciphertext ids, MPC masks
and channel transcripts are charged exactly as that sequence charges them.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .backend import ParameterError, onehot_batch
from .encodings import EncodingKind, PackedMatrix, next_pow2, tile_wave
from .fixedpoint import (FixedPointParams, attention_weights, attention_weights_rows, causal_attention_weights,
                         fp_truncate)
from .linear_kernels import fold_wave
from .nonlinear import (MpcChannel, SharePair, he_to_shares_finish, he_to_shares_start, he_to_shares_wave, reconstruct,
                        share_vector, shares_to_he_wave)

__all__ = ["ScoreLayout", "ScoreVector", "arcc_inner_inner", "arcc_inner_outer", "attention_step",
           "attention_step_heads", "broadcast_slot", "broadcast_wave", "compact_scores", "prefill_attention",
           "prefill_attention_heads"]


class ScoreLayout(Enum):
    PREFILL_ALIGNED = "prefill_aligned"
    BLOCK_ALIGNED = "block_aligned"


@dataclass
class ScoreVector:
    parts: list
    valid_len: int
    layout: ScoreLayout
    block: int | None = None

    @property
    def ct(self):
        return self.parts[0]


def _onehots(n: int, slots):
    """One-hot plaintext masks as a symbolic batch (cached on the device by key)."""
    return onehot_batch(n, slots)


# list of (label, perf_counter) when CGB_HOST_TRACE is set (host timeline of a step)
_TRACE = [] if os.environ.get("CGB_HOST_TRACE") else None


def _mark(label):
    if _TRACE is not None:
        _TRACE.append((label, time.perf_counter()))


def _C(ctx):
    return type(ctx)


# ----------------------------------------------------------------------------
# broadcasts
# ----------------------------------------------------------------------------
def broadcast_wave(wave, js, width: int):
    """Per item: copy slot j to slots [0, width): one-hot mask, rotate j to
    slot 0, ceil(log2 width) doublings (arcc.py:80-94)."""
    C = _C(wave.ctxs[0])
    n = wave.ctxs[0].params.n_slots
    js = np.asarray(js, dtype=np.int64)
    if js.size and (js.min() < 0 or js.max() >= n) or not 1 <= width <= n:
        raise ParameterError(f"slot / width {width} out of range for {n} slots")
    out = C.w_rotate(C.w_mult_plain(wave, _onehots(n, js)), js)
    steps = []
    filled = 1
    while filled < width:
        steps.append(-filled)
        filled *= 2
    if hasattr(C, "w_rotate_add_chain"):
        return C.w_rotate_add_chain(out, steps)
    for st in steps:
        out = C.w_rotate(out, st, add_input=True)
    return out


def broadcast_slot(a, j: int, width: int, ctx):
    n = ctx.params.n_slots
    if not 0 <= j < n or not 1 <= width <= n:
        raise ParameterError(f"slot {j} / width {width} out of range for {n} slots")
    return broadcast_wave(_C(ctx).wave_of([a], [ctx]), [j], width).handles()[0]


# ----------------------------------------------------------------------------
# inner-inner / inner-outer (single query; the decode path uses the head-batched
# schedule in attention_step_heads)
# ----------------------------------------------------------------------------
def arcc_inner_inner(coeffs, basis: PackedMatrix, ctx) -> ScoreVector:
    """sum_j coeffs[j] * vector_j (arcc.py:97-152)."""
    C = _C(ctx)
    n = ctx.params.n_slots
    kind = basis.encoding.kind
    if not basis.encrypted:
        raise ParameterError("inner-inner basis must be encrypted")
    q = C.wave_of([coeffs], [ctx])
    if kind in (EncodingKind.OUTER, EncodingKind.INNER):
        L = len(basis.parts)
        if L == 0 or (kind is EncodingKind.INNER and basis.encoding.rows == 0):
            raise ParameterError("empty basis")
        b = broadcast_wave(q.take(np.zeros(L, np.int64)), np.arange(L), n)
        prods = C.w_mult_cipher(b, C.wave_of(basis.parts, [ctx] * L))
        acc = C.w_sum(prods, [np.arange(L)])
        valid = basis.encoding.rows if kind is EncodingKind.OUTER else basis.encoding.cols
        return ScoreVector(acc.handles(), valid, ScoreLayout.PREFILL_ALIGNED)
    if kind is EncodingKind.INNER_COMPACTED:
        d, rows, B = basis.encoding.cols, basis.encoding.rows, basis.encoding.block
        if rows == 0:
            raise ParameterError("empty basis")
        r = np.arange(rows)
        pieces = broadcast_wave(q.take(np.zeros(rows, np.int64)), r, d)
        bpos = r % B
        moved = np.nonzero(bpos)[0]
        if moved.size:
            rot = C.w_rotate(pieces.take(moved), -(bpos[moved] * d))
            order = np.concatenate([np.nonzero(bpos == 0)[0], moved])
            pieces = type(pieces).concat([pieces.take(np.nonzero(bpos == 0)[0]), rot]).take(np.argsort(order))
        nparts = len(basis.parts)
        cq = C.w_sum(pieces, [np.arange(qi * B, min(rows, (qi + 1) * B)) for qi in range(nparts)])
        prods = C.w_mult_cipher(cq, C.wave_of(basis.parts, [ctx] * nparts))
        acc = C.w_sum(prods, [np.arange(nparts)])
        acc = fold_wave(acc, n // d, first_step=d) if d < n else acc
        return ScoreVector(acc.handles(), d, ScoreLayout.PREFILL_ALIGNED)
    raise ParameterError(f"inner-inner does not accept a {kind} basis")


def arcc_inner_outer(v, rows: PackedMatrix, ctx) -> ScoreVector:
    """<v, row_r>, one score per block start (arcc.py:155-195)."""
    C = _C(ctx)
    n = ctx.params.n_slots
    kind = rows.encoding.kind
    if not rows.encrypted:
        raise ParameterError("inner-outer rows must be encrypted")
    if rows.encoding.rows == 0:
        raise ParameterError("empty row set")
    d = rows.encoding.cols
    nparts = len(rows.parts)
    vw = C.wave_of([v], [ctx])
    if kind is EncodingKind.INNER_COMPACTED:
        vt = tile_wave(vw, d, rows.encoding.block)
        prods = C.w_mult_cipher(vt.take(np.zeros(nparts, np.int64)), C.wave_of(rows.parts, [ctx] * nparts))
        folded = fold_wave(prods, d)
        return ScoreVector(folded.handles(), rows.encoding.rows, ScoreLayout.BLOCK_ALIGNED, block=d)
    if kind is EncodingKind.INNER:
        w = next_pow2(d)
        per_ct = n // w
        prods = C.w_mult_cipher(vw.take(np.zeros(nparts, np.int64)), C.wave_of(rows.parts, [ctx] * nparts))
        dots = fold_wave(prods, w)
        placed = C.w_mult_plain(dots, _onehots(n, np.zeros(nparts, np.int64)))
        b = np.arange(nparts) % per_ct
        moved = np.nonzero(b)[0]
        if moved.size:
            rot = C.w_rotate(placed.take(moved), -(b[moved] * w))
            order = np.concatenate([np.nonzero(b == 0)[0], moved])
            placed = type(placed).concat([placed.take(np.nonzero(b == 0)[0]), rot]).take(np.argsort(order))
        groups = [np.arange(s, min(nparts, s + per_ct)) for s in range(0, nparts, per_ct)]
        parts = C.w_sum(placed, groups)
        return ScoreVector(parts.handles(), rows.encoding.rows, ScoreLayout.BLOCK_ALIGNED, block=w)
    raise ParameterError(f"inner-outer does not accept a {kind} row set")


def compact_scores(s: ScoreVector, ctx) -> ScoreVector:
    """Block-start scores -> contiguous slots (arcc.py:198-214)."""
    C = _C(ctx)
    if s.layout is not ScoreLayout.BLOCK_ALIGNED:
        raise ParameterError("compact_scores expects a block-aligned input")
    n = ctx.params.n_slots
    if s.valid_len > n:
        raise ParameterError("too many scores for one ciphertext")
    per_ct = n // s.block
    r = np.arange(s.valid_len)
    qidx, b = np.divmod(r, per_ct)
    src = b * s.block
    parts = C.wave_of(s.parts, [ctx] * len(s.parts))
    pieces = C.w_mult_plain(parts.take(qidx), _onehots(n, src))
    moved = np.nonzero(src != r)[0]
    if moved.size:
        rot = C.w_rotate(pieces.take(moved), (src - r)[moved])
        stay = np.nonzero(src == r)[0]
        pieces = type(pieces).concat([pieces.take(stay), rot]).take(np.argsort(np.concatenate([stay, moved])))
    acc = C.w_sum(pieces, [r])
    return ScoreVector(acc.handles(), s.valid_len, ScoreLayout.PREFILL_ALIGNED)


def _dot_into_slot(weights_ct, column_ct, slot: int, ctx):
    """mult_cipher, full-width fold, one-hot mask (arcc.py:222-231)."""
    C = _C(ctx)
    n = ctx.params.n_slots
    prod = C.w_mult_cipher(C.wave_of([weights_ct], [ctx]), C.wave_of([column_ct], [ctx]))
    return C.w_mult_plain(fold_wave(prod, n), _onehots(n, [slot])).handles()[0]


def _column_period(P: PackedMatrix, idx: int, period: int, ctx):
    col = P.parts[idx]
    if P.slot_period == period:
        return col
    if P.slot_period is None:
        return tile_wave(_C(ctx).wave_of([col], [ctx]), period, ctx.params.n_slots // period).handles()[0]
    raise ParameterError(f"column padding period {P.slot_period} incompatible with {period}")


# ----------------------------------------------------------------------------
# decode attention, batched over heads
# ----------------------------------------------------------------------------
def attention_step(q, cache, fp: FixedPointParams, ctx, mpc: MpcChannel):
    """One decode-step attention of one head (arcc.py:320-379)."""
    return attention_step_heads([q], [cache], fp, [ctx], [mpc])[0]


HEAD_GROUPS = int(os.environ.get("CGB_HEAD_GROUPS", "2"))


def attention_step_heads(qs, caches, fp: FixedPointParams, ctxs, mpcs, groups: int | None = None) -> list:
    """``attention_step`` for H independent heads in one wave schedule.

    Head h uses context ctxs[h] (its counters, ids and encryption stream)
    and channel mpcs[h] (its masks and transcript), exactly as H sequential
    ``attention_step`` calls would; ctxs may repeat only if the heads would
    have run back to back on that context (then encryptions are assigned in
    head order, which is the sequential order).

    With distinct contexts the heads run as ``groups`` interleaved groups: the
    client side of one group's round trips (decrypt, softmax / truncation,
    re-encrypt) overlaps the device work of the next group, each group's
    decryption waited for on its own.  Every head's op sequence is unchanged."""
    H = len(qs)
    groups = HEAD_GROUPS if groups is None else groups
    if groups <= 1 or H < 2 * groups or len({id(c) for c in ctxs}) < H:
        return _drive([_attention_step_gen(qs, caches, fp, ctxs, mpcs)])[0]
    cuts = np.linspace(0, H, groups + 1).astype(int)
    gens = [_attention_step_gen(qs[a:b], caches[a:b], fp, ctxs[a:b], mpcs[a:b]) for a, b in zip(cuts, cuts[1:])]
    return [o for outs in _drive(gens) for o in outs]


def _drive(gens) -> list:
    """Advance the generators round-robin to completion; their return values."""
    out = [None] * len(gens)
    live = list(range(len(gens)))
    while live:
        for g in list(live):
            try:
                next(gens[g])
            except StopIteration as stop:
                out[g] = stop.value
                live.remove(g)
    return out


def _attention_step_gen(qs, caches, fp: FixedPointParams, ctxs, mpcs):
    """The step of attention_step_heads; yields after enqueueing each client decryption."""
    _mark("step.start")
    H = len(qs)
    c0 = ctxs[0]
    C = _C(c0)
    n, p = c0.params.n_slots, c0.params.plain_modulus
    for cache in caches:
        if cache.m + cache.t_auto == 0:
            raise ParameterError("attention over an empty cache")
    qw = C.wave_of(qs, ctxs)

    # ---- scores: prefill segment (inner-inner over outer-packed K) ------------
    pref_heads = [h for h in range(H) if caches[h].m > 0]
    score_items = []  # (head, wave, length) in per-head reference order
    pref_acc = None
    if pref_heads:
        d2s = [len(caches[h].prefill_K.parts) for h in pref_heads]
        src = np.repeat(np.asarray(pref_heads), d2s)
        js = np.concatenate([np.arange(d) for d in d2s])
        b = broadcast_wave(qw.take(src), js, n)
        kparts = [pt for h in pref_heads for pt in caches[h].prefill_K.parts]
        prods = C.w_mult_cipher(b, C.wave_of(kparts, [ctxs[h] for h in src]), resident_b=True)
        bounds = np.concatenate([[0], np.cumsum(d2s)])
        pref_acc = C.w_sum(prods, [np.arange(bounds[i], bounds[i + 1]) for i in range(len(pref_heads))])
    # ---- scores: generated segment (inner-outer over compacted K) -------------
    auto_heads = [h for h in range(H) if caches[h].t_auto > 0]
    auto_sc = None
    if auto_heads:
        # tile each head's query (same d2 and B for every head of a layer)
        d2, B = caches[auto_heads[0]].d2, caches[auto_heads[0]].B
        vt = tile_wave(qw.take(auto_heads), d2, B)
        nparts = [len(caches[h].auto_K.parts) for h in auto_heads]
        rep = np.repeat(np.arange(len(auto_heads)), nparts)
        kparts = [pt for h in auto_heads for pt in caches[h].auto_K.parts]
        prods = C.w_mult_cipher(vt.take(rep), C.wave_of(kparts, [ctxs[auto_heads[i]] for i in rep]), resident_b=True)
        auto_sc = fold_wave(prods, d2)
    # masked decryption of every score ciphertext, per head in reference order
    order, chans, lens, ap = [], [], [], 0
    pref_pos = {h: i for i, h in enumerate(pref_heads)}
    auto_pos = {}
    for i, h in enumerate(auto_heads):
        auto_pos[h] = (ap, len(caches[h].auto_K.parts))
        ap += len(caches[h].auto_K.parts)
    waves = []
    for h in range(H):
        if h in pref_pos:
            waves.append(("p", pref_pos[h]))
            chans.append(mpcs[h])
            lens.append(caches[h].m)
        if h in auto_pos:
            s, k = auto_pos[h]
            for j in range(k):
                waves.append(("a", s + j))
                chans.append(mpcs[h])
                lens.append(n)
    W = type(qw)
    parts = []
    for kind, idx in waves:
        parts.append((pref_acc if kind == "p" else auto_sc).take([idx]))
    # Every channel draw of this step is known now: score masks, weight re-share,
    # output masks, truncation re-share.  Drawing them while the GPU works on the
    # scores takes the RNG off the two client round trips (same calls, same order).
    plan = [(ch, n) for ch in chans]
    for h in range(H):
        cache = caches[h]
        if cache.m > 0:
            plan.append((mpcs[h], cache.m))
        if cache.t_auto > 0:
            plan.extend((mpcs[h], n) for _ in range(len(cache.auto_V.parts)))
    plan.extend((mpcs[h], n) for h in range(H))
    plan.extend((mpcs[h], caches[h].d2) for h in range(H))
    _mark("scores.enqueued")
    for ch, length in plan:
        ch.predraw([length])
    _mark("masks.predrawn")
    pend = he_to_shares_start(W.concat(parts), chans, lens) if parts else None
    yield
    shares = he_to_shares_finish(pend) if parts else []
    _mark("scores.decrypted")
    # ---- client: reassemble scores, softmax -------------------------------------
    rows, si = [], 0
    for h in range(H):
        cache = caches[h]
        pieces = []
        if cache.m > 0:
            pieces.append(reconstruct(shares[si]))
            si += 1
        for qi in range(len(cache.auto_K.parts) if cache.t_auto > 0 else 0):
            sp = shares[si]
            si += 1
            rows_here = min(cache.B, cache.t_auto - qi * cache.B)
            at = np.arange(rows_here) * cache.d2  # only the block starts carry scores
            pieces.append(reconstruct(SharePair(sp.client[at], sp.server[at], sp.p, rows_here)))
        rows.append(np.concatenate(pieces))
    if len({r.shape[0] for r in rows}) == 1 and len({c.d2 for c in caches}) == 1:
        weights = list(attention_weights_rows(np.stack(rows), caches[0].d2, fp))  # all heads at once
    else:
        weights = [attention_weights(rows[h], caches[h].d2, fp) for h in range(H)]
    for h in range(H):
        mpcs[h].transfer("decode_softmax", caches[h].m + caches[h].t_auto, trips=3 + fp.reciprocal_iters)
    # ---- weights back under encryption: a_pref, then one coefficient ct per auto part
    sp_list, s_ctx, s_ch, s_tag = [], [], [], []
    for h in range(H):
        cache, a = caches[h], weights[h]
        if cache.m > 0:
            sp_list.append(share_vector(a[: cache.m], mpcs[h]))
            s_ctx.append(ctxs[h]); s_ch.append(mpcs[h]); s_tag.append(("p", h, 0))
        if cache.t_auto > 0:
            for qi in range(len(cache.auto_V.parts)):
                rows_here = min(cache.B, cache.t_auto - qi * cache.B)
                seg = a[cache.m + qi * cache.B: cache.m + qi * cache.B + rows_here]
                coeff = np.zeros(n, dtype=np.int64)
                coeff[: rows_here * cache.d2] = np.repeat(seg, cache.d2)
                sp_list.append(share_vector(coeff, mpcs[h]))
                s_ctx.append(ctxs[h]); s_ch.append(mpcs[h]); s_tag.append(("a", h, qi))
    _mark("softmax.done")
    enc = shares_to_he_wave(sp_list, s_ctx, s_ch) if sp_list else None
    _mark("weights.encrypted")
    # ---- values: prefill segment, sum_c dot_into_slot(a_pref, V_c, c) ------------
    o_parts, o_groups = [], []
    pv = None
    if pref_heads:
        a_idx = [i for i, t in enumerate(s_tag) if t[0] == "p"]
        d2s = [len(caches[h].prefill_V.parts) for h in pref_heads]
        rep = np.repeat(np.asarray(a_idx), d2s)
        vparts = [pt for h in pref_heads for pt in caches[h].prefill_V.parts]
        src_heads = np.repeat(np.asarray(pref_heads), d2s)
        prods = C.w_mult_cipher(enc.take(rep), C.wave_of(vparts, [ctxs[h] for h in src_heads]), resident_b=True)
        tot = fold_wave(prods, n)
        cs = np.concatenate([np.arange(d) for d in d2s])
        pieces = C.w_mult_plain(tot, _onehots(n, cs))
        bounds = np.concatenate([[0], np.cumsum(d2s)])
        pv = C.w_sum(pieces, [np.arange(bounds[i], bounds[i + 1]) for i in range(len(pref_heads))])
    av = None
    if auto_heads:
        a_idx = [i for i, t in enumerate(s_tag) if t[0] == "a"]
        vparts = [pt for h in auto_heads for pt in caches[h].auto_V.parts]
        owners = [ctxs[h] for h in auto_heads for _ in caches[h].auto_V.parts]
        prods = C.w_mult_cipher(enc.take(a_idx), C.wave_of(vparts, owners), resident_b=True)
        nparts = [len(caches[h].auto_V.parts) for h in auto_heads]
        bounds = np.concatenate([[0], np.cumsum(nparts)])
        acc = C.w_sum(prods, [np.arange(bounds[i], bounds[i + 1]) for i in range(len(auto_heads))])
        d2 = caches[auto_heads[0]].d2
        av = fold_wave(acc, n // d2, first_step=d2) if d2 < n else acc
    # combine the two segments per head
    outs = []
    for h in range(H):
        if h in pref_pos and h in auto_pos:
            i = pref_pos[h]
            j = auto_heads.index(h)
            outs.append(("both", i, j))
        elif h in pref_pos:
            outs.append(("p", pref_pos[h], None))
        else:
            outs.append(("a", None, auto_heads.index(h)))
    both = [o for o in outs if o[0] == "both"]
    summed = None
    if both:
        summed = C.w_add(pv.take([o[1] for o in both]), av.take([o[2] for o in both]))
    o_list, bi = [], 0
    for kind, i, j in outs:
        if kind == "both":
            o_list.append(summed.take([bi]))
            bi += 1
        elif kind == "p":
            o_list.append(pv.take([i]))
        else:
            o_list.append(av.take([j]))
    ow = W.concat(o_list)
    _mark("values.enqueued")
    # ---- output: masked decrypt (d2 slots), truncate, re-encrypt -----------------
    d2s = [c.d2 for c in caches]
    pend = he_to_shares_start(ow, mpcs, d2s)
    yield
    sh = he_to_shares_finish(pend)
    _mark("values.decrypted")
    tr = [_truncate(s, fp, ch) for s, ch in zip(sh, mpcs)]
    out = shares_to_he_wave(tr, ctxs, mpcs).handles()
    _mark("step.end")
    return out


def _truncate(s: SharePair, fp: FixedPointParams, ch: MpcChannel, mask=None) -> SharePair:
    """nonlinear.truncate with an optional pre-drawn re-share mask."""
    out = fp_truncate(reconstruct(s), fp.f)
    ch.transfer("truncate", s.length, trips=3)
    if mask is None:
        return share_vector(out, ch)
    secret = np.mod(np.asarray(out, dtype=np.int64), ch.p)
    return SharePair((secret - mask) % ch.p, mask, ch.p, secret.shape[0])


# ----------------------------------------------------------------------------
# prefill attention (outer-outer score diagonals), batched over heads
# ----------------------------------------------------------------------------
PREFILL_CHUNK = int(os.environ.get("CGB_PREFILL_CHUNK", "3072"))  # ciphertexts per wave of the sweeps
EXT_A_SWEEP = os.environ.get("CGB_EXT_A", "1") != "0"


def prefill_attention(Q, K, V, fp: FixedPointParams, ctx, mpc: MpcChannel, causal: bool = True) -> PackedMatrix:
    """arcc.py:248-317 for one head."""
    return prefill_attention_heads([Q], [K], [V], fp, [ctx], [mpc], causal)[0]


def prefill_attention_heads(Qs, Ks, Vs, fp: FixedPointParams, ctxs, mpcs, causal: bool = True) -> list:
    """``prefill_attention`` (arcc.py:248-317) for H independent heads, swept
    together: every score-diagonal shift r is ONE batched key switch over all
    heads' K columns (one Galois key for H x d2 ciphertexts), and the value
    sweep's products, folds and one-hot selections run over all heads' columns
    in the same waves.  Head h uses ctxs[h] and mpcs[h] exactly as its own
    prefill_attention call would: its masks are drawn and its transcript
    written in the reference's order, so outputs, ids, counters and transcripts
    equal H sequential calls (tests/test_gpu_hotpath.py)."""
    H = len(Qs)
    c0 = ctxs[0]
    C = _C(c0)
    n, p = c0.params.n_slots, c0.params.plain_modulus
    for Q, K, V in zip(Qs, Ks, Vs):
        for name, P in (("Q", Q), ("K", K), ("V", V)):
            if P.encoding.kind is not EncodingKind.OUTER or not P.encrypted:
                raise ParameterError(f"{name} must be an encrypted outer packing")
        if not (Q.encoding == K.encoding == V.encoding):
            raise ParameterError("Q, K, V disagree on dimensions")
    shapes = {(Q.encoding.rows, Q.encoding.cols, K.slot_period) for Q, K in zip(Qs, Ks)}
    if len(shapes) > 1 or len({id(c) for c in ctxs}) < H:
        # heads of different shapes, or sharing a context (whose draws would interleave):
        # one head at a time
        return [prefill_attention_heads([Qs[h]], [Ks[h]], [Vs[h]], fp, [ctxs[h]], [mpcs[h]], causal)[0]
                for h in range(H)]
    m, d2 = Qs[0].encoding.rows, Qs[0].encoding.cols
    w = next_pow2(m)
    Kw = type(C.wave_of(Ks[0].parts, [ctxs[0]] * d2)).concat(
        [C.wave_of(Ks[h].parts, [ctxs[h]] * d2) for h in range(H)])
    period = Ks[0].slot_period
    if period == w:
        kcols = Kw
    elif period is None:
        kcols = tile_wave(Kw, w, n // w)  # item h d2 + c
    else:
        raise ParameterError(f"column padding period {period} incompatible with {w}")
    Qw = type(Kw).concat([C.wave_of(Qs[h].parts, [ctxs[h]] * d2) for h in range(H)])
    # ---- score diagonals r = 0..w-1: acc_{h,r} = sum_c Q_{h,c} * rot(K_{h,c}, r) ----
    diag_shares = [[] for _ in range(H)]
    rs_per = max(1, PREFILL_CHUNK // (d2 * H))
    for r0 in range(0, w, rs_per):
        rs = np.arange(r0, min(w, r0 + rs_per))
        # items (r, h, c): one shift's H x d2 columns together, one key
        it_r = np.repeat(rs, H * d2)
        it_hc = np.tile(np.arange(H * d2), rs.size)
        nz = np.nonzero(it_r > 0)[0]
        z = np.nonzero(it_r == 0)[0]
        pieces = []
        if z.size:
            pieces.append(kcols.take(it_hc[z]))
        if nz.size:
            pieces.append(C.w_rotate(kcols.take(it_hc[nz]), it_r[nz]))
        order = np.concatenate([z, nz])
        kr = type(kcols).concat(pieces).take(np.argsort(order))
        # Q's columns recur for every row shift: the resident operand (mult_cipher is
        # symmetric word for word -- (a0 b0, a0 b1 + a1 b0, a1 b1) -- and both operands
        # belong to the head's context)
        prods = C.w_mult_cipher(kr, Qw.take(it_hc), resident_b=True)
        groups = [np.arange(g * d2, (g + 1) * d2) for g in range(rs.size * H)]  # group (r, h)
        acc = C.w_sum(prods, groups)
        # he_to_shares per head in r order (each head's channel draws its diagonals in order)
        g_h = np.tile(np.arange(H), rs.size)
        by_head = np.argsort(g_h, kind="stable")  # (h, r) order
        sh = he_to_shares_wave(acc.take(by_head), [mpcs[h] for h in g_h[by_head]], [m] * by_head.size)
        for k, gi in enumerate(by_head):
            diag_shares[g_h[gi]].append(sh[k])
    # ---- client: S from its diagonals, causal softmax per row; rows back encrypted ----
    a_rows, plans = [], []
    i = np.arange(m)
    for h in range(H):
        mpc, ctx = mpcs[h], ctxs[h]
        S = np.zeros((m, m), dtype=np.int64)
        for r, sp in enumerate(diag_shares[h]):
            vals = reconstruct(sp)
            j = (i + r) % w
            ok = j < m
            S[i[ok], j[ok]] = vals[i[ok]]
        A = np.stack([causal_attention_weights(S[k], k, d2, fp) if causal else attention_weights(S[k], d2, fp)
                      for k in range(m)])
        mpc.transfer("prefill_softmax", m * m, trips=3 + fp.reciprocal_iters)
        rows_sp = [share_vector(A[k], mpc) for k in range(m)]
        a_rows.append(shares_to_he_wave(rows_sp, [ctx] * m, [mpc] * m))
        # values: column c gets sum_i dot_into_slot(a_row_i, V_c, i).  The reference
        # draws (he_to_shares: n words, truncate: m words) column by column; the
        # batched sweep pre-draws them in that order
        plans.append([(mpc.sample_mask(n), mpc.sample_mask(m)) for _ in range(d2)])
    Aw = type(a_rows[0]).concat(a_rows)  # item h m + i
    Vw = type(Kw).concat([C.wave_of(Vs[h].parts, [ctxs[h]] * d2) for h in range(H)])  # item h d2 + c
    # every weight row meets all d2 V columns, over several waves: its base-B extension is
    # computed once here and kept with it (mult_cipher_ext2; same words)
    if hasattr(c0, "ring") and EXT_A_SWEEP:
        ring = c0.ring
        # only with headroom: the sweep's own waves need ~3 PREFILL_CHUNK slots at a time
        if ring.free_slots() > 2 * len(Aw) + 8 * PREFILL_CHUNK:
            ring.ext_B(Aw.aids)
    out_parts = [[None] * d2 for _ in range(H)]
    cols_per = max(1, PREFILL_CHUNK // (m * H))
    for c0_ in range(0, d2, cols_per):
        cs = np.arange(c0_, min(d2, c0_ + cols_per))
        # items (h, c, i), group (h, c)
        hc = [(h, c) for h in range(H) for c in cs]
        it_a = np.concatenate([h * m + np.arange(m) for h, c in hc])
        it_v = np.repeat([h * d2 + c for h, c in hc], m)
        it_i = np.tile(np.arange(m), len(hc))
        prods = C.w_mult_cipher(Aw.take(it_a), Vw.take(it_v), resident_b=True)
        tot = fold_wave(prods, n)
        pieces = C.w_mult_plain(tot, _onehots(n, it_i))
        acc = C.w_sum(pieces, [np.arange(k * m, (k + 1) * m) for k in range(len(hc))])
        # he_to_shares with the planned masks, then truncate / re-encrypt
        r = np.stack([plans[h][c][0] for h, c in hc])
        masked = C.w_add_plain(acc, (p - r) % p, one_shot=True)
        client = C.w_decrypt(masked)
        trs = []
        for k, (h, c) in enumerate(hc):
            mpcs[h].transfer("he_to_shares", n)
            sp = SharePair(client[k, :m].copy(), r[k, :m].copy(), p, m)
            trs.append(_truncate(sp, fp, mpcs[h], mask=plans[h][c][1]))
        hs = shares_to_he_wave(trs, [ctxs[h] for h, _ in hc], [mpcs[h] for h, _ in hc], record=False).handles()
        for k, (h, c) in enumerate(hc):
            out_parts[h][c] = hs[k]
        for h in range(H):
            _reorder_transcript(mpcs[h], cs.size, n)
    return [PackedMatrix(Qs[h].encoding, out_parts[h], encrypted=True, slot_period=None) for h in range(H)]


def _reorder_transcript(mpc: MpcChannel, k: int, n: int):
    """Per column the reference records he_to_shares, truncate, shares_to_he;
    the chunked sweep recorded k x (he_to_shares, truncate) pairs -- append
    each column's shares_to_he right after its pair."""
    tail = mpc.transcript[-2 * k:]
    del mpc.transcript[-2 * k:]
    for i in range(k):
        mpc.transcript.extend(tail[2 * i: 2 * i + 2])
        mpc.transfer("shares_to_he", n)
