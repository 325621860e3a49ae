"""Decoder-layer pipeline over the batched hot path (BASELINE config 3).

Restates the encrypted pipeline of /root/reference/pkg/src/cryptogen/model.py
-- ``prefill`` (:425-497), ``decode_step`` (:500-566), ``generate`` (:569+)
and their helpers ``_matrix_roundtrip`` / ``_vector_roundtrip`` /
``_trunc_packed`` / ``_channels`` (:357-396) -- with the per-head loops run
as waves: the 12 heads' projections, truncation round trips, cache appends,
refreshes and attention steps are batched calls of this package, so every
rotation amount of a head-step is one key switch over all heads.

Semantics kept from the reference: the op sequence per context (counters and
ledger budgets), the channels (one per (layer, head) plus "common", seeded
as model.py:388-398), the client-side fixed-point arithmetic (truncation,
GELU, LayerNorm, softmax) and hence every decrypted value: the generated
tokens and logits equal the reference's.  Mask draws and transcript entries
follow the reference's per-op order within every channel (``_trunc_wave``
draws and records item by item), so share values, masks and transcripts equal
the reference's too (tests/test_layer.py pins them).

Out of the reference: a vocab-50257 unembedding cannot be
diagonal-packed at n = 8192; here a vocabulary wider than n is unembedded in
n-column blocks (``_logits``), and ``unembed_vocab`` can still cap the
unembedded columns while token embeddings keep the full vocabulary.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field, replace

import numpy as np

from .arcc import attention_step_heads, prefill_attention_heads
from .backend import ParameterError
from .encodings import EncodingKind, PackedMatrix, encode
from .fixedpoint import FixedPointParams, fp_gelu, fp_layernorm_rows, fp_truncate, to_signed
from .kv_cache import append_token_heads, init_cache, maybe_refresh_heads
from .linear_kernels import cpmm_outer_diagonal, cpvm_inner_diagonal, cpvm_inner_diagonal_heads
from .nonlinear import (MpcChannel, SharePair, _pool, he_to_shares_wave, host_buffer, neg_mod, reconstruct, share_vector,
                        shares_to_he_wave)

__all__ = ["GenerationState", "Model", "ModelConfig", "decode_step", "generate", "gpt2_layer_model", "prefill"]

_MATS = ("wq", "wk", "wv", "wo", "w1", "w2")
_VECS = ("b1", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")


@dataclass(frozen=True)
class ModelConfig:
    """model.py:58-90; ``unembed_vocab`` columns of the unembedding are computed."""

    layers: int
    d1: int
    heads: int
    ffn_dim: int
    vocab: int
    max_seq: int
    f: int = 8
    unembed_vocab: int | None = None

    def __post_init__(self):
        if min(self.layers, self.d1, self.heads, self.ffn_dim, self.vocab, self.max_seq) < 1:
            raise ParameterError("all model dimensions must be positive")
        if self.d1 % self.heads:
            raise ParameterError(f"d1 = {self.d1} must be divisible by heads = {self.heads}")

    @property
    def d2(self) -> int:
        return self.d1 // self.heads

    @property
    def out_vocab(self) -> int:
        return self.vocab if self.unembed_vocab is None else min(self.vocab, self.unembed_vocab)


@dataclass
class Model:
    config: ModelConfig
    weights: dict  # name -> signed int64 array at scale f (model.py:94-122 naming)
    _diag: dict = field(default_factory=dict, repr=False)

    def layer(self, l: int, name: str) -> np.ndarray:
        return self.weights[f"layer{l}.{name}"]

    def head_slice(self, l: int, name: str, h: int) -> np.ndarray:
        d2 = self.config.d2
        return self.layer(l, name)[:, h * d2:(h + 1) * d2]

    def diag(self, key: str, matrix: np.ndarray, ctx) -> PackedMatrix:
        """Plaintext diagonal packing of a weight, memoized per modulus (model.py:114-122)."""
        tag = (key, ctx.params.n_slots, ctx.params.plain_modulus)
        got = self._diag.get(tag)
        if got is None:
            got = self._diag[tag] = encode(matrix, EncodingKind.DIAGONAL, ctx, encrypted=False)
        return got

    def unembed(self) -> np.ndarray:
        return self.weights["unembed"][:, :self.config.out_vocab]

    def fixed_point(self, ctx) -> FixedPointParams:
        return FixedPointParams(self.config.f, ctx.params.plain_modulus)


def gpt2_layer_model(config: ModelConfig, seed: int = 0, std: float = 0.02) -> Model:
    """GPT-2 initialisation at scale f: weights and
    embeddings round(N(0, std) 2^f), LayerNorm gains 2^f, biases 0."""
    c = config
    rng = np.random.default_rng(np.random.SeedSequence([0x6E7, seed]))
    q = lambda shape: np.round(rng.normal(0.0, std, shape) * (1 << c.f)).astype(np.int64)
    w = {"tok_emb": q((c.vocab, c.d1)), "pos_emb": q((c.max_seq, c.d1))}
    for l in range(c.layers):
        shapes = {"wq": (c.d1, c.d1), "wk": (c.d1, c.d1), "wv": (c.d1, c.d1), "wo": (c.d1, c.d1),
                  "w1": (c.d1, c.ffn_dim), "w2": (c.ffn_dim, c.d1)}
        for k in _MATS:
            w[f"layer{l}.{k}"] = q(shapes[k])
        w[f"layer{l}.b1"] = np.zeros(c.ffn_dim, np.int64)
        w[f"layer{l}.b2"] = np.zeros(c.d1, np.int64)
        for k in ("ln1", "ln2"):
            w[f"layer{l}.{k}_g"] = np.full(c.d1, 1 << c.f, np.int64)
            w[f"layer{l}.{k}_b"] = np.zeros(c.d1, np.int64)
    w["unembed"] = q((c.d1, c.out_vocab))
    return Model(config, w)


@dataclass
class GenerationState:
    position: int
    caches: list  # [layer][head] -> KVCache
    next_logits: np.ndarray
    tokens: list = field(default_factory=list)


def channels(ctx_seed: int, layers: int, heads: int, p: int) -> dict:
    """One channel per (layer, head) plus "common", spawned as model.py:388-398."""
    kids = np.random.SeedSequence([0x707, ctx_seed]).spawn(layers * heads + 1)
    chans = {(l, h): MpcChannel(p, kids[l * heads + h]) for l in range(layers) for h in range(heads)}
    chans["common"] = MpcChannel(p, kids[-1])
    return chans


def _embed(model: Model, token: int, pos: int) -> np.ndarray:
    c = model.config
    if not 0 <= token < c.vocab:
        raise ParameterError(f"token {token} out of vocabulary")
    if pos >= c.max_seq:
        raise ParameterError(f"position {pos} beyond max_seq {c.max_seq}")
    return model.weights["tok_emb"][token] + model.weights["pos_emb"][pos]


# ----------------------------------------------------------------------------
# client round trips, one wave per call
# ----------------------------------------------------------------------------
def _C(ctx):
    return type(ctx)


def _trunc_wave(wave, lengths, fp, ctxs, chans):
    """Per item: he_to_shares -> truncate -> shares_to_he (model.py:370-375,
    :526-531), as one wave.  The reference runs the three steps item by item, so
    each channel draws (n words for the masked decryption, then `length` words
    for the truncation's re-share) and records (he_to_shares, truncate,
    shares_to_he) per item; the masks are drawn and the transcript written in
    exactly that order here, so every share, mask and transcript entry equals
    the per-op code's."""
    C = type(wave.ctxs[0])
    params = wave.ctxs[0].params
    n, p = params.n_slots, params.plain_modulus
    lengths = [int(x) for x in lengths]
    r_dec, r_tr = _draw_in_order(chans, [(n, L) for L in lengths])
    masked = C.w_add_plain(wave, neg_mod(r_dec, p), one_shot=True, canonical=True)
    client = C.w_decrypt(masked)
    shares = []
    for i, (ch, L) in enumerate(zip(chans, lengths)):
        v = client[i, :L] + r_dec[i, :L]  # reconstruct: both shares in [0, p)
        v = np.where(v >= p, v - p, v)
        out = np.mod(fp_truncate(to_signed(v, p), fp.f), p)
        d = out - r_tr[i]
        d[d < 0] += p
        shares.append(SharePair(d, r_tr[i], p, L))
        ch.transfer("he_to_shares", n)
        ch.transfer("truncate", L, trips=3)
        ch.transfer("shares_to_he", n)
    return shares_to_he_wave(shares, ctxs, chans, record=False)


def _draw_in_order(chans, plan):
    """Item i draws plan[i] = (a, b): a words, then b words, from chans[i]; each
    channel's items in list order (its sequence of per-op draws), distinct
    channels on parallel host threads.  Returns (rows of a words, list of b-word arrays)."""
    a = plan[0][0] if plan else 0
    first = host_buffer((len(chans), a))
    second = [None] * len(chans)
    groups = {}
    for i, ch in enumerate(chans):
        groups.setdefault(id(ch), (ch, []))[1].append(i)

    def fill(item):
        ch, idx = item
        for i in idx:
            first[i] = ch.sample_mask(plan[i][0])
            second[i] = ch.sample_mask(plan[i][1])

    if len(groups) > 1 and len(chans) * a >= (1 << 20):
        list(_pool().map(fill, groups.values()))
    else:
        for item in groups.values():
            fill(item)
    return first, second


def _vector_roundtrips(wave, lengths, ctxs, chans, fns):
    """Per item: decrypt through shares, apply fn, re-encrypt (model.py:368-370)."""
    sp = he_to_shares_wave(wave, chans, lengths)
    shares = [share_vector(fn(reconstruct(s)), ch) for s, ch, fn in zip(sp, chans, fns)]
    return shares_to_he_wave(shares, ctxs, chans)


def _matrix_roundtrip(parts, m, ctx, ch, fn):
    """Outer columns -> client matrix (m x d) -> fn -> columns (model.py:357-366)."""
    C = _C(ctx)
    d = len(parts)
    sp = he_to_shares_wave(C.wave_of(parts, [ctx] * d), [ch] * d, [m] * d)
    out = fn(np.stack([reconstruct(s) for s in sp], axis=1))
    shares = [share_vector(out[:, j], ch) for j in range(out.shape[1])]
    return shares_to_he_wave(shares, [ctx] * len(shares), [ch] * len(shares)).handles()


def _logits(model, x_ct, ctx, fp):
    """model.py:487-495 / :548-556.  A vocabulary wider than the slot count (the
    reference raises there) is unembedded in n-column blocks, one
    CPVM per block over copies of the same activation: every block rotates it by
    the same n - 1 steps, so the rotations are one hoisted key switch per step
    (content classes, backend.Wave) and each block only adds its products,
    block by block (serial_products) so they fit the ciphertext arena."""
    c = model.config
    p, n = ctx.params.plain_modulus, ctx.params.n_slots
    V = c.out_vocab
    if V <= n:
        ct = cpvm_inner_diagonal(x_ct, model.diag("unembed", model.unembed(), ctx), ctx)
        return fp_truncate(to_signed(ctx.decrypt(ct), p)[:V], fp.f)
    nb = -(-V // n)
    Ws = []
    for b in range(nb):
        W = model._diag.get((f"unembed.{b}", n, p))
        if W is None:  # block b: columns b n .. (b + 1) n - 1, zero past the vocabulary
            blk = np.zeros((c.d1, n), np.int64)
            cols = model.unembed()[:, b * n:min(V, (b + 1) * n)]
            blk[:, :cols.shape[1]] = cols
            W = model.diag(f"unembed.{b}", blk, ctx)
        Ws.append(W)
    # UNEMBED_GROUP blocks share one rotation wave; their products run block by block
    cts = []
    for b0 in range(0, nb, UNEMBED_GROUP):
        k = min(UNEMBED_GROUP, nb - b0)
        cts += cpvm_inner_diagonal_heads([x_ct] * k, Ws[b0:b0 + k], [ctx] * k, serial_products=True)
    vals = np.concatenate([to_signed(ctx.decrypt(ct), p) for ct in cts])
    return fp_truncate(vals[:V], fp.f)


# slot blocks of a wide unembedding per batched CPVM (their products share the arena)
UNEMBED_GROUP = int(os.environ.get("CGB_UNEMBED_GROUP", "8"))


# ----------------------------------------------------------------------------
# prefill (model.py:425-497)
# ----------------------------------------------------------------------------
def prefill(model: Model, prompt: list, ctx, chans=None) -> GenerationState:
    c = model.config
    if not 1 <= len(prompt) <= c.max_seq:
        raise ParameterError("prompt length out of range")
    C = _C(ctx)
    p, n = ctx.params.plain_modulus, ctx.params.n_slots
    fp = model.fixed_point(ctx)
    chans = channels(0, c.layers, c.heads, p) if chans is None else chans
    m = len(prompt)
    X = np.stack([_embed(model, t, i) for i, t in enumerate(prompt)])
    X_enc = encode(np.mod(X, p), EncodingKind.OUTER, ctx)
    caches = [[None] * c.heads for _ in range(c.layers)]
    for l in range(c.layers):
        hctxs = [ctx.fork() for _ in range(c.heads)]
        hch = [chans[(l, h)] for h in range(c.heads)]
        # projections, then one truncation wave over the 3 x heads x d2 columns
        # (per channel: Q columns, K columns, V columns -- the reference's order)
        proj = {}
        for h in range(c.heads):
            for name in ("wq", "wk", "wv"):
                W = model.diag(f"{l}.{name}.{h}", model.head_slice(l, name, h), hctxs[h])
                proj[(h, name)] = cpmm_outer_diagonal(X_enc, W, hctxs[h])
        items, ictx, ich, lens = [], [], [], []
        for h in range(c.heads):
            for name in ("wq", "wk", "wv"):
                P = proj[(h, name)]
                items += P.parts
                ictx += [hctxs[h]] * len(P.parts)
                ich += [hch[h]] * len(P.parts)
                lens += [P.encoding.rows] * len(P.parts)
        tr = _trunc_wave(C.wave_of(items, ictx), lens, fp, ictx, ich).handles()
        del items  # the raw projections' ciphertexts are released here (arena headroom)
        mats, k = {}, 0
        for h in range(c.heads):
            for name in ("wq", "wk", "wv"):
                P = proj[(h, name)]
                mats[(h, name)] = PackedMatrix(P.encoding, tr[k:k + len(P.parts)], encrypted=True, slot_period=None)
                k += len(P.parts)
        Qs, Ks, Vs = ([mats[(h, nm)] for h in range(c.heads)] for nm in ("wq", "wk", "wv"))
        del proj, mats, tr
        Os = prefill_attention_heads(Qs, Ks, Vs, fp, hctxs, hch, causal=True)
        del Qs
        o_parts = []
        for h in range(c.heads):
            ctx.join(hctxs[h])
            caches[l][h] = init_cache(Ks[h], Vs[h], hctxs[h])
            o_parts.extend(Os[h].parts)
        O_cat = PackedMatrix(replace(X_enc.encoding, cols=c.d1), o_parts, encrypted=True, slot_period=None)
        del Os, o_parts

        ch = chans["common"]
        attn = cpmm_outer_diagonal(O_cat, model.diag(f"{l}.wo", model.layer(l, "wo"), ctx), ctx)
        del O_cat
        attn = _trunc_wave(C.wave_of(attn.parts, [ctx] * c.d1), [m] * c.d1, fp, [ctx] * c.d1, [ch] * c.d1).handles()
        resid = C.w_add(C.wave_of(X_enc.parts, [ctx] * c.d1), C.wave_of(attn, [ctx] * c.d1)).handles()
        g1, b1 = model.layer(l, "ln1_g"), model.layer(l, "ln1_b")
        del attn
        ln1 = _matrix_roundtrip(resid, m, ctx, ch, lambda M: fp_layernorm_rows(M, g1, b1, fp))
        del resid
        X_enc = PackedMatrix(replace(X_enc.encoding, cols=c.d1), ln1, encrypted=True)

        h1 = cpmm_outer_diagonal(X_enc, model.diag(f"{l}.w1", model.layer(l, "w1"), ctx), ctx)
        h1p = _bias_parts(h1.parts, model.layer(l, "b1") << fp.f, m, ctx)
        del h1
        hact = _matrix_roundtrip(h1p, m, ctx, ch, lambda M: fp_gelu(fp_truncate(M, fp.f), fp))
        del h1p
        Hm = PackedMatrix(replace(X_enc.encoding, cols=c.ffn_dim), hact, encrypted=True)

        h2 = cpmm_outer_diagonal(Hm, model.diag(f"{l}.w2", model.layer(l, "w2"), ctx), ctx)
        del Hm, hact
        h2p = _bias_parts(h2.parts, model.layer(l, "b2") << fp.f, m, ctx)
        del h2
        h2t = _matrix_roundtrip(h2p, m, ctx, ch, lambda M: fp_truncate(M, fp.f))
        del h2p
        resid2 = C.w_add(C.wave_of(ln1, [ctx] * c.d1), C.wave_of(h2t, [ctx] * c.d1)).handles()
        g2, b2 = model.layer(l, "ln2_g"), model.layer(l, "ln2_b")
        ln2 = _matrix_roundtrip(resid2, m, ctx, ch, lambda M: fp_layernorm_rows(M, g2, b2, fp))
        X_enc = PackedMatrix(replace(X_enc.encoding, cols=c.d1), ln2, encrypted=True)

    # last position's row back through shares, logits via the decode-side CPVM (model.py:487-495)
    ch = chans["common"]
    sp = he_to_shares_wave(C.wave_of(X_enc.parts, [ctx] * c.d1), [ch] * c.d1, [m] * c.d1)
    last = np.array([reconstruct(s)[m - 1] for s in sp])
    x_last = shares_to_he_wave([share_vector(last, ch)], [ctx], [ch]).handles()[0]
    return GenerationState(position=m, caches=caches, next_logits=_logits(model, x_last, ctx, fp),
                           tokens=list(prompt))


def _bias_parts(parts, bias_f, m, ctx):
    """Column j += bias_f[j] on its m live slots (model.py:477-480, :486-489)."""
    C = _C(ctx)
    p, n = ctx.params.plain_modulus, ctx.params.n_slots
    vecs = np.zeros((len(parts), n), np.int64)
    vecs[:, :m] = np.mod(np.asarray(bias_f, np.int64), p)[:, None]
    return C.w_add_plain(C.wave_of(parts, [ctx] * len(parts)), vecs, one_shot=True).handles()


# ----------------------------------------------------------------------------
# decode (model.py:500-566)
# ----------------------------------------------------------------------------
def decode_step(model: Model, state: GenerationState, ctx, chans=None, force_refresh: bool = False):
    """Greedy token from state.next_logits, then one single-token pass.
    ``force_refresh`` refreshes every cache part first (config 3's "noise
    refresh each step"); otherwise the reference's lazy check runs."""
    c = model.config
    C = _C(ctx)
    p = ctx.params.plain_modulus
    fp = model.fixed_point(ctx)
    chans = channels(0, c.layers, c.heads, p) if chans is None else chans
    token = int(np.argmax(state.next_logits))
    pos = state.position
    if pos >= c.max_seq:
        raise ParameterError("generation exceeded max_seq")
    caches = [maybe_refresh_heads(state.caches[l], [ctx] * c.heads, [chans[(l, h)] for h in range(c.heads)],
                                  force=force_refresh) for l in range(c.layers)]
    x = ctx.encrypt(ctx.plain_from_dense(np.mod(_embed(model, token, pos), p)))
    for l in range(c.layers):
        hctxs = [ctx.fork() for _ in range(c.heads)]
        hch = [chans[(l, h)] for h in range(c.heads)]
        Ws, ictx, ich = [], [], []
        for h in range(c.heads):
            for name in ("wq", "wk", "wv"):
                Ws.append(model.diag(f"{l}.{name}.{h}", model.head_slice(l, name, h), hctxs[h]))
                ictx.append(hctxs[h])
                ich.append(hch[h])
        raw = cpvm_inner_diagonal_heads([x] * len(Ws), Ws, ictx)
        qkv = _trunc_wave(C.wave_of(raw, ictx), [c.d2] * len(raw), fp, ictx, ich).handles()
        qs, ks, vs = qkv[0::3], qkv[1::3], qkv[2::3]
        cs = append_token_heads(caches[l], ks, vs, hctxs)
        outs = attention_step_heads(qs, cs, fp, hctxs, hch)
        for h in range(c.heads):
            ctx.join(hctxs[h])
            caches[l][h] = cs[h]
        # o_cat = oh_0 + rotate(oh_h, -h d2) ... (model.py:539-543)
        if c.heads > 1:
            rot = C.w_rotate(C.wave_of(outs[1:], [ctx] * (c.heads - 1)), -c.d2 * np.arange(1, c.heads))
            allw = type(rot).concat([C.wave_of(outs[:1], [ctx]), rot])
            o_cat = C.w_sum(allw, [np.arange(c.heads)]).handles()[0]
        else:
            o_cat = outs[0]
        ch = chans["common"]
        attn = cpvm_inner_diagonal(o_cat, model.diag(f"{l}.wo", model.layer(l, "wo"), ctx), ctx)
        attn = _trunc_wave(C.wave_of([attn], [ctx]), [c.d1], fp, [ctx], [ch]).handles()[0]
        g1, b1 = model.layer(l, "ln1_g"), model.layer(l, "ln1_b")
        x = _vector_roundtrips(C.wave_of([ctx.add(x, attn)], [ctx]), [c.d1], [ctx], [ch],
                               [lambda v: fp_layernorm_rows(v[None, :], g1, b1, fp)[0]]).handles()[0]
        h1 = cpvm_inner_diagonal(x, model.diag(f"{l}.w1", model.layer(l, "w1"), ctx), ctx)
        h1 = ctx.add_plain(h1, ctx.plain_from_dense(np.mod(model.layer(l, "b1") << fp.f, p)))
        h1 = _vector_roundtrips(C.wave_of([h1], [ctx]), [c.ffn_dim], [ctx], [ch],
                                [lambda v: fp_gelu(fp_truncate(v, fp.f), fp)]).handles()[0]
        h2 = cpvm_inner_diagonal(h1, model.diag(f"{l}.w2", model.layer(l, "w2"), ctx), ctx)
        h2 = ctx.add_plain(h2, ctx.plain_from_dense(np.mod(model.layer(l, "b2") << fp.f, p)))
        h2 = _vector_roundtrips(C.wave_of([h2], [ctx]), [c.d1], [ctx], [ch],
                                [lambda v: fp_truncate(v, fp.f)]).handles()[0]
        g2, b2 = model.layer(l, "ln2_g"), model.layer(l, "ln2_b")
        x = _vector_roundtrips(C.wave_of([ctx.add(x, h2)], [ctx]), [c.d1], [ctx], [ch],
                               [lambda v: fp_layernorm_rows(v[None, :], g2, b2, fp)[0]]).handles()[0]
    new = GenerationState(position=pos + 1, caches=caches, next_logits=_logits(model, x, ctx, fp),
                          tokens=state.tokens + [token])
    return token, new


def generate(model: Model, prompt: list, k: int, ctx, force_refresh: bool = False):
    """Encrypted prefill + k greedy decode steps (model.py:569+); returns the
    generated tokens and the final state."""
    c = model.config
    if not 1 <= len(prompt) <= c.max_seq or len(prompt) + k > c.max_seq:
        raise ParameterError("prompt/generation length exceeds max_seq")
    chans = channels(0, c.layers, c.heads, ctx.params.plain_modulus)
    state = prefill(model, prompt, ctx, chans)
    out = []
    for _ in range(k):
        tok, state = decode_step(model, state, ctx, chans, force_refresh=force_refresh)
        out.append(tok)
    return out, state
