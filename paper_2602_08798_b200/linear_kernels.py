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

import numpy as np

from .backend import ParameterError
from .encodings import Encoding, EncodingKind, PackedMatrix, decode, next_pow2

__all__ = ["cpmm_outer_diagonal", "cpvm_inner_diagonal", "fold_sum", "fold_wave"]


def _fold_checks(block: int, n: int):
    if block < 1 or block > n or block & (block - 1) or n % block:
        raise ParameterError(f"block {block} must be a power of two dividing {n}")


def fold_wave(wave, block: int, first_step: int = 1):
    """Per item: slot i <- a[i] + ... + a[i + block - 1] (cyclic), by
    log2(block) batched rotate-and-add steps 1, 2, 4, ...  (:27-42)."""
    C = type(wave.ctxs[0])
    _fold_checks(block, wave.ctxs[0].params.n_slots)
    step = first_step
    while step < block * first_step:
        wave = C.w_rotate(wave, step, add_input=True)
        step *= 2
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
    C = type(ctx)
    Wv = _diagonal_weights(W, ctx)
    d1, d2 = W.encoding.rows, W.encoding.cols
    n = ctx.params.n_slots
    wd1, wd2 = next_pow2(d1), next_pow2(d2)
    wp = max(wd1, wd2)
    if wp > n:
        raise ParameterError(f"operand width {wp} exceeds {n} slots")
    xw = C.wave_of([x], [ctx])
    if wp != n:
        xw = C.w_rotate(xw, -wp, add_input=True)
    # generalized diagonals k = 0 .. wd2-1 as one plaintext batch
    j = np.arange(wp)
    col = j % wd2
    pts = np.zeros((wd2, n), dtype=np.int64)
    for k in range(wd2):
        row = (j + k) % wp
        ok = (row < d1) & (col < d2)
        pts[k, :wp][ok] = Wv[row[ok], col[ok]]
    if wd2 > 1:
        rot = C.w_rotate(xw.take(np.zeros(wd2 - 1, np.int64)), np.arange(1, wd2))
        xs = type(xw).concat([xw, rot])
    else:
        xs = xw
    prods = C.w_mult_plain(xs, pts)
    acc = C.w_sum(prods, [np.arange(wd2)])
    return fold_wave(acc, wp // wd2, first_step=wd2).handles()[0] if wp > wd2 else acc.handles()[0]


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
        cs = range(c0, min(d2, c0 + chunk))
        pts = np.zeros((len(cs) * ng, n), dtype=np.int64)
        for ci, c in enumerate(cs):
            for gi, g in enumerate(starts):
                row = pts[ci * ng + gi]
                for u in range(min(group, d1 - g)):
                    row[u * w: u * w + m] = Wv[g + u, c]
        prods = C.w_mult_plain(work.take(np.tile(np.arange(ng), len(cs))), pts, one_shot=chunk < d2)
        prods = fold_wave(prods, group, first_step=w) if group > 1 else prods
        out += C.w_sum(prods, [np.arange(ci * ng, (ci + 1) * ng) for ci in range(len(cs))]).handles()
    return PackedMatrix(Encoding(EncodingKind.OUTER, m, d2), out, encrypted=True, slot_period=w)


CPMM_CHUNK = 4096  # plaintext products per wave of cpmm_outer_diagonal
