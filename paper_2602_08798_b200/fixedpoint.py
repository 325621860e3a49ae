"""Signed fixed-point helpers the attention path calls on the client side.

Out of the B200 scope proper (the MPC non-linear protocols stay host code),
but ``attention_step`` / ``prefill_attention`` need the reference's integer
softmax between the score and value phases, so the pieces on that path are
restated here from /root/reference/pkg/src/cryptogen/fixedpoint.py:
embedding and truncation (:86-106), Newton reciprocal (:131-145), softmax
(:148-175) and the attention-weight wrappers (:204-221).  The polynomial
constants are the reference's frozen fit (fixedpoint.py:51-53).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .backend import ParameterError

# exp(r) on (-ln2, 0] as c2 r^2 + c1 r + c0 (reference fit, fixedpoint.py:51-53)
EXP_COEFFS = (0.3558034634, 0.9634474169, 0.9982613301)
SHIFT_CAP = 48
CAUSAL_MASK_EXPONENT = 6


@dataclass(frozen=True)
class FixedPointParams:
    f: int
    p: int
    reciprocal_iters: int = 4

    def __post_init__(self):
        if self.f < 1:
            raise ParameterError("fraction bits must be positive")
        if (1 << (2 * self.f + 6)) >= self.p:
            raise ParameterError(f"need 2^(2f+6) < p for product headroom; f={self.f} p={self.p}")
        if self.reciprocal_iters < 1:
            raise ParameterError("reciprocal needs at least one iteration")

    @property
    def scale(self) -> int:
        return 1 << self.f

    def quantize(self, v: float) -> int:
        return int(round(v * self.scale))


def to_signed(v, p: int):
    v = np.asarray(v, dtype=np.int64)
    return np.where(v > p // 2, v - p, v)


def from_signed(v, p: int):
    v = np.asarray(v, dtype=np.int64)
    if v.size and v.min() > -p and v.max() < p:  # the usual case: one conditional add, no modulo
        return np.where(v < 0, v + p, v)
    return np.mod(v, p)


def fp_encode(x, fp: FixedPointParams) -> np.ndarray:
    return np.round(np.asarray(x, dtype=np.float64) * fp.scale).astype(np.int64)


def fp_decode(v, fp: FixedPointParams) -> np.ndarray:
    return np.asarray(v, dtype=np.float64) / fp.scale


def fp_truncate(v, f: int):
    return np.asarray(v, dtype=np.int64) >> f


def fp_reciprocal(s: int, fp: FixedPointParams, work_bits: int | None = None):
    """Newton iteration y <- y (2 - s y) from the bit-length lower bound."""
    if s <= 0:
        raise ParameterError("reciprocal needs a positive input")
    q = 2 * fp.f if work_bits is None else work_bits
    y = 1 << max(0, fp.f + q - int(s).bit_length())
    two = 1 << (q + 1)
    for _ in range(fp.reciprocal_iters):
        y = (y * (two - ((s * y) >> fp.f))) >> q
    return y, q


def fp_softmax(s, fp: FixedPointParams) -> np.ndarray:
    """Integer softmax: x = s - max = -ln2 z + r, e = poly(r) >> z, normalise."""
    f = fp.f
    s = np.asarray(s, dtype=np.int64)
    if s.shape[0] == 0:
        raise ParameterError("softmax needs at least one score")
    if s.shape[0] == 1:
        return np.array([fp.scale], dtype=np.int64)
    c2, c1, c0 = (fp.quantize(c) for c in EXP_COEFFS)
    x = s - s.max()
    z = ((-x) * fp.quantize(1.0 / math.log(2.0))) >> (2 * f)
    r = x + z * fp.quantize(math.log(2.0))
    poly = np.maximum(((c2 * ((r * r) >> f)) >> f) + ((c1 * r) >> f) + c0, 0)
    e = poly >> np.minimum(z, SHIFT_CAP)
    rec, q = fp_reciprocal(int(e.sum()), fp)
    return (e * rec + (1 << (q - 1))) >> q


def fp_softmax_rows(S, fp: FixedPointParams) -> np.ndarray:
    """fp_softmax of every row of S (rows of one length), vectorised over rows.

    Same integer operations as fp_softmax row by row; the Newton reciprocal runs
    on int64 vectors, exact while every intermediate stays below 2^62 (checked:
    rows whose exponent sum could overflow fall back to the per-row path)."""
    f = fp.f
    S = np.asarray(S, dtype=np.int64)
    if S.ndim != 2 or S.shape[1] <= 1:
        return np.stack([fp_softmax(row, fp) for row in S]) if len(S) else S
    c2, c1, c0 = (fp.quantize(c) for c in EXP_COEFFS)
    x = S - S.max(axis=1, keepdims=True)
    z = ((-x) * fp.quantize(1.0 / math.log(2.0))) >> (2 * f)
    r = x + z * fp.quantize(math.log(2.0))
    poly = np.maximum(((c2 * ((r * r) >> f)) >> f) + ((c1 * r) >> f) + c0, 0)
    e = poly >> np.minimum(z, SHIFT_CAP)
    tot = e.sum(axis=1)
    q = 2 * f
    if tot.min() <= 0 or int(tot.max()).bit_length() + f + q > 61 or 3 * q + 2 * f > 61:
        return np.stack([fp_softmax(row, fp) for row in S])
    bits = np.frexp(tot.astype(np.float64))[1].astype(np.int64)  # bit length (tot < 2^53: exact)
    y = np.left_shift(np.int64(1), np.maximum(0, f + q - bits))
    two = np.int64(1) << (q + 1)
    for _ in range(fp.reciprocal_iters):
        y = (y * (two - ((tot * y) >> f))) >> q
    return (e * y[:, None] + (np.int64(1) << (q - 1))) >> q


def attention_weights_rows(S_2f, d2: int, fp: FixedPointParams) -> np.ndarray:
    """attention_weights of every row of S_2f (one head per row)."""
    return fp_softmax_rows(_scaled_scores(S_2f, d2, fp), fp)


def _scaled_scores(scores_2f, d2: int, fp: FixedPointParams) -> np.ndarray:
    s1 = fp_truncate(np.asarray(scores_2f, dtype=np.int64), fp.f)
    return (s1 * fp.quantize(1.0 / math.sqrt(d2))) >> fp.f


def attention_weights(scores_2f, d2: int, fp: FixedPointParams) -> np.ndarray:
    """scale-2f scores -> softmax(s / sqrt(d2)) at scale f (fixedpoint.py:204-209)."""
    return fp_softmax(_scaled_scores(scores_2f, d2, fp), fp)


def causal_attention_weights(row_2f, row_index: int, d2: int, fp: FixedPointParams) -> np.ndarray:
    """Prefill row with the additive causal mask -2^(f+6) (fixedpoint.py:212-221)."""
    s2 = _scaled_scores(row_2f, d2, fp)
    s2[row_index + 1:] -= 1 << (fp.f + CAUSAL_MASK_EXPONENT)
    return fp_softmax(s2, fp)


# ----------------------------------------------------------------------------
# client-side activations of the decoder layer (BASELINE config 3 harness)
# ----------------------------------------------------------------------------
# GELU on [0, 3.2] as c4 (x^2 + beta x)^2 + c2' x^2 + c1 x (the reference's
# frozen quartic, fixedpoint.py:43-49); beta = c3 / (2 c4), c2' = c2 - c4 beta^2
GELU_CLIP = 3.2
_GELU_C = (0.0203101927, -0.1792823041, 0.5309976652, 0.4701539873)  # c4, c3, c2, c1


def fp_gelu(x, fp: FixedPointParams) -> np.ndarray:
    """GELU on signed scale-f integers, elementwise (fixedpoint.py:109-128):
    the quartic on |x| <= clip, GELU(x) = x + GELU(-x) for x < 0, identity /
    zero beyond the clip."""
    c4f, c3f, c2f, c1f = _GELU_C
    beta_f = c3f / (2.0 * c4f)
    f = fp.f
    x = np.asarray(x, dtype=np.int64)
    clip = fp.quantize(GELU_CLIP)
    c4, beta, c2p, c1 = (fp.quantize(v) for v in (c4f, beta_f, c2f - c4f * beta_f * beta_f, c1f))
    ax = np.minimum(np.abs(x), clip)
    sq = (ax * ax) >> f
    u = sq + ((beta * ax) >> f)
    g = ((c4 * ((u * u) >> f)) >> f) + ((c2p * sq) >> f) + ((c1 * ax) >> f)
    near = np.where(x >= 0, g, x + g)
    far = np.where(x > 0, x, 0)
    return np.where(np.abs(x) > clip, far, near)


def _div_round(a: np.ndarray, d: int) -> np.ndarray:
    """Round-half-away-from-zero a / d for int64 arrays (fixedpoint.py:194-198)."""
    a = np.asarray(a, dtype=np.int64)
    pos = (2 * a + d) // (2 * d)
    neg = -((2 * (-a) + d) // (2 * d))
    return np.where(a >= 0, pos, neg)


def fp_layernorm_rows(X, gain, bias, fp: FixedPointParams) -> np.ndarray:
    """LayerNorm of every row of X (signed scale-f), Newton inverse square
    root seeded from the integer square root, 3 iterations
    (fixedpoint.py:178-191, :224-243); a zero-variance row yields the bias."""
    f = fp.f
    X = np.atleast_2d(np.asarray(X, dtype=np.int64))
    gain = np.asarray(gain, dtype=np.int64)
    bias = np.asarray(bias, dtype=np.int64)
    d = X.shape[1]
    if d < 2:
        raise ParameterError("layernorm needs at least two values")
    mu = _div_round(X.sum(axis=1), d)
    c = X - mu[:, None]
    var = _div_round((c * c).sum(axis=1), d)  # scale 2f
    seed = np.array([math.isqrt(int(v)) for v in var], dtype=np.int64)
    y = (np.int64(1) << (2 * f)) // np.maximum(seed, 1)
    three = np.int64(3) << f
    for _ in range(3):
        t = (((var * y) >> (2 * f)) * y) >> f
        y = (y * (three - t)) >> (f + 1)
    out = ((gain[None, :] * ((c * y[:, None]) >> f)) >> f) + bias[None, :]
    out[var == 0] = bias
    return out


def fp_layernorm(x, gain, bias, fp: FixedPointParams) -> np.ndarray:
    """One vector (fixedpoint.py:224-243)."""
    return fp_layernorm_rows(np.asarray(x)[None, :], gain, bias, fp)[0]
