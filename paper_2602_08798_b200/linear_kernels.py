"""CT x PT projections and the rotate-and-add fold they share, batched.

Mirrors /root/reference/pkg/src/cryptogen/linear_kernels.py: ``fold_sum``
(:27-42), the prefill CPMM over outer-packed activations (:51-102) and the
decode CPVM over a diagonal weight (:105-142).  Every independent chain of
the reference loops is one item of a wave, so e.g. the wd2 rotations of the
CPVM are a single batched key switch and the d2 x groups plaintext products
of the CPMM are one launch.  Logical op counts, ledger budgets and
ciphertext words equal the reference op sequence's.
"""

from __future__ import annotations

import itertools

import numpy as np

from .backend import ParameterError, PlainBatch
from .encodings import Encoding, EncodingKind, PackedMatrix, decode, next_pow2

__all__ = ["cpmm_outer_diagonal", "cpvm_inner_diagonal", "cpvm_inner_diagonal_heads", "fold_sum", "fold_wave"]


def _fold_checks(block: int, n: int):
    if block < 1 or block > n or block & (block - 1) or n % block:
        raise ParameterError(f"block {block} must be a power of two dividing {n}")


def fold_wave(wave, block: int, first_step: int = 1):
    """Per item: slot i <- a[i] + ... + a[i + block - 1] (cyclic), by
    log2(block) batched rotate-and-add steps 1, 2, 4, ...  (:27-42)."""
    C = type(wave.ctxs[0])
    _fold_checks(block, wave.ctxs[0].params.n_slots)
    steps = []
    step = first_step
    while step < block * first_step:
        steps.append(step)
        step *= 2
    if hasattr(C, "w_rotate_add_chain"):  # one library call for the whole chain (same words and ledger)
        return C.w_rotate_add_chain(wave, steps)
    for step in steps:
        wave = C.w_rotate(wave, step, add_input=True)
    return wave


def fold_sum(a, block: int, ctx):
    C = type(ctx)
    return fold_wave(C.wave_of([a], [ctx]), block).handles()[0]


def _diagonal_weights(W: PackedMatrix, ctx) -> np.ndarray:
    if W.encrypted or W.encoding.kind is not EncodingKind.DIAGONAL:
        raise ParameterError("weights must be a plaintext diagonal PackedMatrix")
    return decode(W, ctx)


def cpvm_inner_diagonal(x, W: PackedMatrix, ctx):
    """x (inner, length d1) times diagonal plaintext W (d1 x d2) -> slots [0, d2)."""
    return cpvm_inner_diagonal_heads([x], [W], [ctx])[0]


def cpvm_inner_diagonal_heads(xs, Ws, ctxs, serial_products: bool = False) -> list:
    """``cpvm_inner_diagonal`` for B independent (x, W, ctx) triples of one
    shape (e.g. the 3 x 12 per-head decode projections, model.py:521-526):
    each rotation amount is one batched key switch over all B items; item i's
    ops are charged to ctxs[i] exactly as its own call would charge them."""
    B = len(xs)
    C = type(ctxs[0])
    for W in Ws:
        if W.encrypted or W.encoding.kind is not EncodingKind.DIAGONAL:
            raise ParameterError("weights must be a plaintext diagonal PackedMatrix")
    d1, d2 = Ws[0].encoding.rows, Ws[0].encoding.cols
    if any((W.encoding.rows, W.encoding.cols) != (d1, d2) for W in Ws):
        raise ParameterError("batched cpvm needs one weight shape")
    n, p = ctxs[0].params.n_slots, ctxs[0].params.plain_modulus
    wd1, wd2 = next_pow2(d1), next_pow2(d2)
    wp = max(wd1, wd2)
    if wp > n:
        raise ParameterError(f"operand width {wp} exceeds {n} slots")
    # the dense weight is decoded only the first time a weight is seen
    Wv = [None if _diagonal_rows(W, None, n, p, wd2, wp)[1] is not None else _diagonal_weights(W, c)
          for W, c in zip(Ws, ctxs)]
    xw = C.wave_of(xs, ctxs)
    if wp != n:
        xw = C.w_rotate(xw, -wp, add_input=True)
    # generalized diagonals k = 0 .. wd2-1 of each weight: built once per weight and
    # named symbolically, so the device plaintext cache keeps them across steps
    rows = {}
    for W, wv in zip(Ws, Wv):
        uid, r = _diagonal_rows(W, wv, n, p, wd2, wp)
        rows[uid] = r
    uids = [_diagonal_rows(W, None, n, p, wd2, wp)[0] for W in Ws]

    def build(keys):
        return np.stack([rows[k[1]][k[4]] for k in keys])

    key = lambda b, k: ("cpvm", uids[b], n, p, k)
    if wd2 > 1:
        rot = C.w_rotate(xw.take(np.repeat(np.arange(B), wd2 - 1)), np.tile(np.arange(1, wd2), B))
        xs_w = type(xw).concat([xw, rot])
        # item b: [b, B + b (wd2 - 1) .. B + (b + 1)(wd2 - 1) - 1] <-> diagonals 0 .. wd2-1
        keys = [key(b, 0) for b in range(B)] + [key(b, k) for b in range(B) for k in range(1, wd2)]
        groups = [np.concatenate([[b], B + b * (wd2 - 1) + np.arange(wd2 - 1)]) for b in range(B)]
    else:
        xs_w, keys, groups = xw, [key(b, 0) for b in range(B)], [np.array([b]) for b in range(B)]
    if serial_products:
        # one item's products at a time (same words; the rotations above stay one
        # wave): a wide unembedding's 7 x 8192 products never coexist in the arena
        accs = []
        for g in groups:
            prods = C.w_mult_plain(xs_w.take(g), PlainBatch([keys[i] for i in g], build))
            accs.append(C.w_sum(prods, [np.arange(g.size)]))
        acc = type(xw).concat(accs)
    else:
        prods = C.w_mult_plain(xs_w, PlainBatch(keys, build))
        acc = C.w_sum(prods, groups)
    return (fold_wave(acc, wp // wd2, first_step=wd2) if wp > wd2 else acc).handles()


_uids = itertools.count()


def _diagonal_rows(W: PackedMatrix, Wv, n: int, p: int, wd2: int, wp: int):
    """(uid, residues[wd2, n]) of W's generalized diagonals: row k holds
    W[(j + k) mod wp, j mod wd2] at slot j (linear_kernels.py:105-142)."""
    cache = W.__dict__.setdefault("_cpvm_rows", {})
    uid = W.__dict__.setdefault("_cpvm_uid", next(_uids))
    got = cache.get((n, p))
    if got is None and Wv is not None:
        d1, d2 = Wv.shape
        j = np.arange(wp)
        col = j % wd2
        got = np.zeros((wd2, n), dtype=np.int64)
        for k in range(wd2):
            row = (j + k) % wp
            ok = (row < d1) & (col < d2)
            got[k, :wp][ok] = Wv[row[ok], col[ok]]
        got = np.mod(got, p)
        cache[(n, p)] = got
    return uid, got


def cpmm_outer_diagonal(X: PackedMatrix, W: PackedMatrix, ctx) -> PackedMatrix:
    """Outer-packed X (m x d1) times diagonal plaintext W (d1 x d2); columns
    stacked n / next_pow2(m) per working ciphertext (:51-102)."""
    C = type(ctx)
    if X.encoding.kind is not EncodingKind.OUTER or not X.encrypted:
        raise ParameterError("cpmm expects an encrypted outer-packed activation")
    if X.slot_period is not None:
        raise ParameterError("cpmm expects zero-padded input columns")
    Wv = _diagonal_weights(W, ctx)
    m, d1 = X.encoding.rows, X.encoding.cols
    if d1 != W.encoding.rows:
        raise ParameterError(f"dimension mismatch: X is {m}x{d1}, W is {W.encoding.rows}x{W.encoding.cols}")
    d2 = W.encoding.cols
    n = ctx.params.n_slots
    w = next_pow2(m)
    if w > n:
        raise ParameterError(f"{m} rows do not fit {n} slots")
    group = n // w
    starts = list(range(0, d1, group))
    Xw = C.wave_of(X.parts, [ctx] * d1)
    # stack columns g+u (u >= 1) rotated right by u*w onto column g
    src = [g + u for g in starts for u in range(1, min(group, d1 - g))]
    amt = [-(u * w) for g in starts for u in range(1, min(group, d1 - g))]
    rot = C.w_rotate(Xw.take(src), amt) if src else None
    pieces = [Xw.take(starts)] + ([rot] if rot is not None else [])
    allw = type(Xw).concat(pieces)
    groups, pos, ri = [], len(starts), 0
    for gi, g in enumerate(starts):
        k = min(group, d1 - g) - 1
        groups.append(np.concatenate([[gi], np.arange(pos + ri, pos + ri + k)]).astype(np.int64))
        ri += k
    work = C.w_sum(allw, groups)
    # one plaintext product per (output column c, working ct g), column-major; wide
    # outputs (e.g. the 768 x 3072 FFN projection: 36864 products) go in column
    # chunks of at most CPMM_CHUNK products so the products' ciphertexts stay a few
    # GB -- every column's chain is independent, so its words are unchanged
    ng = len(starts)
    chunk = max(1, CPMM_CHUNK // ng) if d2 * ng > CPMM_CHUNK else d2
    out = []
    for c0 in range(0, d2, chunk):
        cs = np.arange(c0, min(d2, c0 + chunk))
        # row (ci, gi): W[g_gi + u, c] on the m live slots of block u (zero past d1)
        Wpad = np.zeros((ng * group, d2), dtype=np.int64)
        Wpad[:d1] = Wv
        blocks = Wpad[:, cs].reshape(ng, group, len(cs)).transpose(2, 0, 1)  # [ci][gi][u]
        pts = np.zeros((len(cs), ng, group, w), dtype=np.int64)
        pts[..., :m] = blocks[..., None]
        # projection weights are used once per call: encoded as scratch plaintexts
        prods = C.w_mult_plain(work.take(np.tile(np.arange(ng), len(cs))), pts.reshape(len(cs) * ng, n),
                               one_shot=True)
        prods = fold_wave(prods, group, first_step=w) if group > 1 else prods
        out += C.w_sum(prods, [np.arange(ci * ng, (ci + 1) * ng) for ci in range(len(cs))]).handles()
    return PackedMatrix(Encoding(EncodingKind.OUTER, m, d2), out, encrypted=True, slot_period=w)


CPMM_CHUNK = 4096  # plaintext products per wave of cpmm_outer_diagonal
