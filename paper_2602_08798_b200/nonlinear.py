"""HE <-> additive-share conversion on the hot path (server-side masking).

Restates the conversion half of /root/reference/pkg/src/cryptogen/
nonlinear.py: the channel's byte/round ledger and mask RNG (:63-93),
``share_vector`` (:101-106), ``he_to_shares`` (:112-125), ``shares_to_he``
(:128-137) and ``truncate`` (:140-144).  The MPC protocols themselves
(GELU / softmax / layernorm over shares) are host code outside this tier.

Parity-critical: masks are drawn from ``MpcChannel.rng`` with exactly the
reference's lengths and order (he_to_shares always draws n words, even for
shorter shares).  The batched forms below take one channel per item and
draw item by item, which is the order the per-op code would draw in.
"""

from __future__ import annotations

import collections
import json
import os
from dataclasses import dataclass

import numpy as np

from .backend import ParameterError
from .fixedpoint import FixedPointParams, fp_truncate, from_signed, to_signed

__all__ = ["MpcChannel", "SharePair", "he_to_shares", "he_to_shares_finish", "he_to_shares_start", "he_to_shares_wave",
           "reconstruct", "share_vector",
           "shares_to_he", "shares_to_he_wave", "truncate"]


@dataclass
class SharePair:
    client: np.ndarray
    server: np.ndarray
    p: int
    length: int

    def __post_init__(self):
        if self.client.shape != (self.length,) or self.server.shape != (self.length,):
            raise ParameterError("share arrays must match the declared length")


class MpcChannel:
    """Bytes/rounds tally plus the mask RNG of one serial conversation."""

    def __init__(self, p: int, seed=0):
        self.p = p
        self.word_bits = p.bit_length()
        self.bytes_sent = 0
        self.rounds = 0
        ss = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
        self.rng = np.random.default_rng(ss)
        self.transcript: list = []
        self._pre = collections.deque()  # masks drawn ahead of use, in draw order

    def vector_bytes(self, elements: int) -> int:
        return elements * self.word_bits // 8

    def transfer(self, op: str, elements: int, trips: int = 1) -> None:
        nbytes = trips * self.vector_bytes(elements)
        self.bytes_sent += nbytes
        self.rounds += trips
        self.transcript.append({"op": op, "elements": elements, "trips": trips, "bytes": nbytes})

    def sample_mask(self, length: int) -> np.ndarray:
        if self._pre:
            r = self._pre.popleft()
            if r.shape[0] != length:
                raise RuntimeError(f"pre-drawn mask of {r.shape[0]} words, {length} requested: "
                                   "the draw sequence diverged from the predraw plan")
            return r
        return self.rng.integers(0, self.p, size=length, dtype=np.int64)

    def predraw(self, lengths) -> None:
        """Draw the next masks now (same generator calls, same order) so a
        later ``sample_mask`` is off the critical path; the masks, and so
        every share and ciphertext, are unchanged."""
        for n in lengths:
            self._pre.append(self.rng.integers(0, self.p, size=int(n), dtype=np.int64))

    def transcript_json(self) -> str:
        return json.dumps({"bytes_sent": self.bytes_sent, "rounds": self.rounds, "log": self.transcript}, indent=2)


_POOL = None
_PINNED = None


# page-locked buffers up to 128 MB: the per-step round trips (a decode step's forced
# refresh moves 100 MB each way) reuse them from torch's caching host allocator;
# larger one-off batches (a prefill's 3072-column round trips) stay pageable, where
# allocating fresh page-locked memory would cost more than the copies it saves
PINNED_MAX_WORDS = int(os.environ.get("CGB_PINNED_MAX_MB", "128")) << 17


def host_buffer(shape, min_words: int = 1 << 16) -> np.ndarray:
    """An int64 host array, page-locked when a CUDA device is present (so its
    upload is a DMA, not a driver-staged copy); plain numpy otherwise."""
    global _PINNED
    if _PINNED is None:
        try:
            import torch

            _PINNED = bool(torch.cuda.is_available())
        except Exception:  # pragma: no cover - torch is part of the image
            _PINNED = False
    if _PINNED and min_words <= int(np.prod(shape)) <= PINNED_MAX_WORDS:
        import torch

        return torch.empty(tuple(shape), dtype=torch.int64, pin_memory=True).numpy()
    return np.empty(shape, np.int64)


def _pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _POOL = ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1))
    return _POOL


def neg_mod(r: np.ndarray, p: int) -> np.ndarray:
    """(-r) mod p for r in [0, p), without an integer modulo, into a host buffer;
    large batches (a forced refresh negates 1.5k x 8192 words) in row blocks on
    the host threads (numpy releases the GIL)."""
    out = host_buffer(r.shape)

    def neg(sl):
        o = out[sl]
        np.subtract(p, r[sl], out=o)
        hit = o == p
        if hit.any():
            o[hit] = 0

    if r.ndim == 2 and r.shape[0] >= 16 and r.size >= (1 << 21):
        step = -(-r.shape[0] // 8)
        list(_pool().map(neg, [slice(i, i + step) for i in range(0, r.shape[0], step)]))
    else:
        neg(slice(None))
    return out


def draw_masks(chans, n: int) -> np.ndarray:
    """rows[i] = chans[i].sample_mask(n), each channel's draws in item order (its
    sequence is unchanged); distinct channels draw on parallel host threads (the
    generator fill releases the GIL) when there is enough to draw."""
    global _POOL
    out = host_buffer((len(chans), n))
    groups = {}
    for i, ch in enumerate(chans):
        groups.setdefault(id(ch), (ch, []))[1].append(i)

    def fill(item):
        ch, idx = item
        for i in idx:
            out[i] = ch.sample_mask(n)

    if len(groups) > 1 and len(chans) * n >= (1 << 20):
        list(_pool().map(fill, groups.values()))
    else:
        for item in groups.values():
            fill(item)
    return out


DEVICE_MASKS = os.environ.get("CGB_DEVICE_MASKS", "1") != "0"
_M64 = (1 << 64) - 1


def _pcg_state_words(ch: "MpcChannel") -> list:
    st = ch.rng.bit_generator.state
    if st["bit_generator"] != "PCG64":
        raise ParameterError("device masks reproduce numpy's PCG64 only")
    s, inc = st["state"]["state"], st["state"]["inc"]
    return [s >> 64, s & _M64, inc >> 64, inc & _M64, int(st["has_uint32"]), int(st["uinteger"])]


def device_masks_ok(chans) -> bool:
    """Whether these channels' next masks can be drawn on the device: numpy PCG64
    generators with no masks pre-drawn on the host (those come first)."""
    return DEVICE_MASKS and all(not ch._pre and type(ch.rng.bit_generator).__name__ == "PCG64" for ch in chans)


def device_masks(ring, chans, want_neg: bool = True, want_pos: bool = True, want_masks: bool = False):
    """Item i's mask = chans[i].sample_mask(n_slots), drawn on the device
    (cgb_mask_pcg64: numpy's PCG64 + bounded-integer sampling, bit-exact) and
    encoded as add_plain plaintexts of t - r (neg) and r (pos); each channel's
    generator continues exactly where the host draws would have left it.
    Returns (pt_neg, pt_pos, masks or None); the caller frees the plaintexts."""
    uniq, idx = [], {}
    chan_of = np.empty(len(chans), np.int32)
    for i, ch in enumerate(chans):
        k = idx.get(id(ch))
        if k is None:
            k = idx[id(ch)] = len(uniq)
            uniq.append(ch)
        chan_of[i] = k
    st = np.array([_pcg_state_words(ch) for ch in uniq], dtype=np.uint64)
    neg = ring.alloc_pt(len(chans)) if want_neg else None
    pos = ring.alloc_pt(len(chans)) if want_pos else None
    masks = ring.mask_pcg64(chan_of, st, neg, pos, want_masks)
    for ch, w in zip(uniq, st.tolist()):
        bg = ch.rng.bit_generator
        s = bg.state
        s["state"]["state"] = (int(w[0]) << 64) | int(w[1])
        s["has_uint32"], s["uinteger"] = int(w[4]), int(w[5])
        bg.state = s
    return neg, pos, masks


def reconstruct(s: SharePair) -> np.ndarray:
    v = s.client + s.server
    if v.size and v.min() >= 0 and v.max() < 2 * s.p:  # both shares in [0, p): one conditional subtract
        v = np.where(v >= s.p, v - s.p, v)
    else:
        v = v % s.p
    return to_signed(v, s.p)


def share_vector(values, ch: MpcChannel) -> SharePair:
    secret = from_signed(values, ch.p)
    r = ch.sample_mask(secret.shape[0])
    d = secret - r  # both in [0, p): (secret - r) mod p is one conditional add
    d[d < 0] += ch.p
    return SharePair(d, r, ch.p, secret.shape[0])


def truncate(s: SharePair, fp: FixedPointParams, ch: MpcChannel) -> SharePair:
    """Floor-divide the reconstruction by 2^f and re-share (nonlinear.py:140-144)."""
    out = fp_truncate(reconstruct(s), fp.f)
    ch.transfer("truncate", s.length, trips=3)
    return share_vector(out, ch)


# ----------------------------------------------------------------------------
# batched conversions: one wave of ciphertexts, one channel per item
# ----------------------------------------------------------------------------
def he_to_shares_wave(wave, chans, lengths) -> list:
    """Server masks each ciphertext with a fresh r (n words from its channel),
    the client decrypts; returns one SharePair per item."""
    return he_to_shares_finish(he_to_shares_start(wave, chans, lengths))


def he_to_shares_start(wave, chans, lengths):
    """he_to_shares_wave up to the client's decryption, which is enqueued, not
    awaited: masks drawn and masked ciphertexts formed in the same order."""
    C = type(wave.ctxs[0])
    params = wave.ctxs[0].params
    n, p = params.n_slots, params.plain_modulus
    lengths = list(lengths)
    for L in lengths:
        if not 0 < L <= n:
            raise ParameterError(f"share length {L} out of range")
    r = draw_masks(chans, n)
    masked = C.w_add_plain(wave, neg_mod(r, p), one_shot=True, canonical=True)
    return C, C.w_decrypt_start(masked), r, list(chans), lengths, n, p


def he_to_shares_finish(pending) -> list:
    C, dec, r, chans, lengths, n, p = pending
    client = C.w_decrypt_finish(dec)
    out = []
    for i, ch in enumerate(chans):
        ch.transfer("he_to_shares", n)
        L = lengths[i]
        out.append(SharePair(client[i, :L].copy(), r[i, :L].copy(), p, L))
    return out


def shares_to_he_wave(shares, ctxs, chans, record: bool = True):
    """Client encrypts its share, server adds its own; returns a wave.
    ``record=False`` leaves the transcript entries to the caller."""
    c0 = ctxs[0]
    C = type(c0)
    n = c0.params.n_slots
    # shares are residues in [0, p) (share_vector / reconstruct); zero-padded to n slots
    client = np.zeros((len(shares), n), np.int64)
    server = np.zeros((len(shares), n), np.int64)
    for i, sh in enumerate(shares):
        if sh.client.shape[0] > n:
            raise ParameterError("vector longer than slot count")
        client[i, : sh.client.shape[0]] = sh.client
        server[i, : sh.server.shape[0]] = sh.server
    enc = C.w_encrypt(ctxs, client, canonical=True)
    out = C.w_add_plain(enc, server, one_shot=True, canonical=True)
    if record:
        for ch in chans:
            ch.transfer("shares_to_he", n)
    return out


def he_to_shares(ct, ctx, ch: MpcChannel, length: int | None = None) -> SharePair:
    """nonlinear.py:112-125 (one item of the batched form)."""
    n = ctx.params.n_slots
    C = type(ctx)
    return he_to_shares_wave(C.wave_of([ct], [ctx]), [ch], [n if length is None else length])[0]


def shares_to_he(s: SharePair, ctx, ch: MpcChannel):
    """nonlinear.py:128-137 (one item of the batched form)."""
    return shares_to_he_wave([s], [ctx], [ch]).handles()[0]
