"""Drop-in HE substrate: the reference ``Context`` API over the B200 ring.

Reference boundary: ``cryptogen.backend`` (/root/reference/pkg/src/
cryptogen/backend.py).  The reference realises a ciphertext as an n-slot
vector over Z_p with a bit ledger (backend.py:216-230, :295-301) and op
counters (:173-213); this module keeps the ledger and counters byte-for-byte
and replaces the arithmetic with real RNS-BFV ciphertexts that live in the
device arena of ``libcgb200.so``:

  reference                      here
  ---------------------------    ----------------------------------------
  BackendParams / NoiseCosts     same dataclasses, same validation
  OpCounter                      same fields, merge/snapshot/delta/to_json
  SlotCiphertext (:216)          GpuCiphertext: arena id + budget + id
  Context (:245)                 GpuContext: same methods, plus the
                                 batched "wave" API (``Wave``) the fused
                                 hot path in arcc/kv_cache/linear_kernels uses
  new_context (:367)             new_context -> GpuContext (no CPU path)

Layouts: when p = 1 (mod 4n) the ring degree is
N = 2n and the n logical slots are one hypercube row, so a cyclic shift by
k is the single automorphism X -> X^(5^k); otherwise (small test
parameters with p = 1 mod 2n only) N = n and the shift is composed from the
two row automorphisms and two 0/1 masks.

Keys are shared by every context with equal parameters (contexts in the
reference interoperate whenever ``params`` compare equal, backend.py:290);
encryption randomness is per context: ChaCha20 keyed from the context's
SeedSequence, one nonce per encryption in call order.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import os
import threading
import weakref
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as nat

__all__ = [
    "BackendParams", "Context", "DecryptionFailure", "GpuCiphertext", "GpuContext", "NoiseBudgetExhausted",
    "NoiseCosts", "OpCounter", "ParameterError", "PlainVector", "SlotCiphertext", "PlainBatch", "Wave", "default_plain_modulus", "onehot_batch",
    "is_prime", "key_seed", "new_context", "ring_for", "set_key_seed",
]

PlainVector = np.ndarray
MAX_PLAIN_MODULUS = 1 << 31


# ----------------------------------------------------------------------------
# errors and parameters (restating backend.py:45-170)
# ----------------------------------------------------------------------------
class ParameterError(ValueError):
    """Parameters, shapes or ciphertext ownership are invalid (backend.py:45)."""


class NoiseBudgetExhausted(RuntimeError):
    """The ledger would go negative (backend.py:49, :295-301)."""


class DecryptionFailure(RuntimeError):
    """Decryption of a ciphertext whose ledger is at zero (backend.py:53, :312)."""


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (same contract as backend.py:60)."""
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for b in small:
        if n % b == 0:
            return n == b
    d, r = n - 1, 0
    while not d & 1:
        d >>= 1
        r += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def default_plain_modulus(n_slots: int, min_bits: int = 29) -> int:
    """Smallest prime >= 2^min_bits that is 1 mod 2*n_slots (backend.py:84-93)."""
    step = 2 * n_slots
    c = (1 << min_bits) + (-(1 << min_bits) + 1) % step
    while not is_prime(c):
        c += step
    return c


@dataclass(frozen=True)
class NoiseCosts:
    """Ledger cost in bits of each operation (backend.py:96-113)."""

    mult_plain: int = 20
    mult_cipher: int = 40
    rotate: int = 2
    add: int = 0
    add_plain: int = 0

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in ("mult_plain", "mult_cipher", "rotate", "add", "add_plain")}


@dataclass(frozen=True)
class BackendParams:
    """Slot count, plaintext modulus and ledger (backend.py:116-170)."""

    n_slots: int = 8192
    plain_modulus: int = 536903681
    initial_noise_budget: int = 190
    noise_costs: NoiseCosts = field(default_factory=NoiseCosts)
    refresh_threshold: int = 60

    def __post_init__(self):
        n, p = self.n_slots, self.plain_modulus
        if n < 2 or n & (n - 1):
            raise ParameterError(f"n_slots must be a power of two >= 2, got {n}")
        if not is_prime(p):
            raise ParameterError(f"plain_modulus {p} is not prime")
        if p % (2 * n) != 1:
            raise ParameterError(f"plain_modulus {p} must be 1 mod 2*n_slots (= {2 * n})")
        if p >= MAX_PLAIN_MODULUS:
            raise ParameterError(f"plain_modulus {p} exceeds 2^31")
        if any(v < 0 for v in self.noise_costs.as_dict().values()):
            raise ParameterError(f"noise costs must be >= 0, got {self.noise_costs.as_dict()}")
        if not 0 <= self.refresh_threshold < self.initial_noise_budget:
            raise ParameterError("refresh_threshold must lie in [0, initial_noise_budget)")

    @property
    def modulus_bits(self) -> int:
        return self.plain_modulus.bit_length()

    def ciphertext_bytes(self) -> int:
        """Modelled wire size of one ciphertext transfer (backend.py:152-154)."""
        return self.n_slots * self.modulus_bits // 8

    def to_json(self) -> str:
        d = {"n_slots": self.n_slots, "plain_modulus": self.plain_modulus,
             "initial_noise_budget": self.initial_noise_budget, "noise_costs": self.noise_costs.as_dict(),
             "refresh_threshold": self.refresh_threshold}
        return json.dumps(d, indent=2, sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "BackendParams":
        d = json.loads(text)
        return cls(noise_costs=NoiseCosts(**d.pop("noise_costs", {})), **d)


_COUNTER_FIELDS = ("mult_plain", "mult_cipher", "rotate", "add", "add_plain", "encrypt", "decrypt",
                   "refresh_events", "mpc_bytes")


@dataclass
class OpCounter:
    """Monotone per-op tallies (backend.py:173-213)."""

    mult_plain: int = 0
    mult_cipher: int = 0
    rotate: int = 0
    add: int = 0
    add_plain: int = 0
    encrypt: int = 0
    decrypt: int = 0
    refresh_events: int = 0
    mpc_bytes: int = 0

    _FIELDS = _COUNTER_FIELDS

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in _COUNTER_FIELDS}

    def merge(self, other: "OpCounter") -> None:
        for k in _COUNTER_FIELDS:
            setattr(self, k, getattr(self, k) + getattr(other, k))

    def snapshot(self) -> "OpCounter":
        return OpCounter(**self.as_dict())

    def delta(self, since: "OpCounter") -> dict:
        return {k: getattr(self, k) - getattr(since, k) for k in _COUNTER_FIELDS}

    def to_json(self) -> str:
        return json.dumps(self.as_dict(), indent=2, sort_keys=True)


def _params_key(params) -> tuple:
    c = params.noise_costs
    return (params.n_slots, params.plain_modulus)


# ----------------------------------------------------------------------------
# rings: one per (n_slots, p, limbs, key seed), shared by all contexts
# ----------------------------------------------------------------------------
def _default_key_seed() -> int:
    """The keyring seed: CGB_KEY_SEED when set (reproducible runs: tests, benches),
    else a per-process secret from the OS CSPRNG -- the secret and evaluation keys
    are never a function of a public constant."""
    env = os.environ.get("CGB_KEY_SEED")
    return int(env) if env is not None else int.from_bytes(os.urandom(8), "little")


_KEY_SEED = _default_key_seed()
_rings: dict = {}


def set_key_seed(seed: int) -> None:
    """Explicit keyring: contexts created from now on use keys derived from
    ``seed`` (contexts with equal params and the same keyring interoperate, as
    the reference's contexts do, backend.py:290; earlier contexts keep theirs)."""
    global _KEY_SEED
    _KEY_SEED = int(seed)


def key_seed() -> int:
    return _KEY_SEED
_rings_lock = threading.Lock()


def default_limbs(ring_degree: int) -> int:
    """Q limbs of 60 bits.

    N >= 16384 (the production n = 8192 ring): 3 limbs of 49 bits, Q = 147
    bits.  The deepest intermediates of the hot path (decode scores/values
    after one-hot mult_plain + 14 rotations + mult_cipher + 64-term sums;
    prefill P.V columns) keep >= 28 bits of real noise budget (61 with 60-bit
    primes; profiles/r01/params_sweep.md; tests/test_gpu_hotpath.py asserts
    >= 20).  Smaller
    production-size rings get 4 limbs, toy rings 8 (their composite two-row
    rotations spend more real noise per logical op).  CGB_LIMBS overrides."""
    env = os.environ.get("CGB_LIMBS")
    if env:
        return int(env)
    if ring_degree >= 16384:
        return 3
    return 4 if ring_degree >= 2048 else 8


def ring_layout(n_slots: int, p: int) -> tuple[int, bool]:
    """(log2 N, one_row) for a parameter set."""
    if p % (4 * n_slots) == 1:
        return (2 * n_slots).bit_length() - 1, True
    return n_slots.bit_length() - 1, False


def default_qbits(ring_degree: int) -> int:
    """Bit size of the primes (CGB_QBITS overrides).

    Rings of degree >= 4096 use primes < 2^49 so their NTTs run on the FP64
    pipe (exact error-free transformations; 1.2x the integer-pipe NTT per
    transform, 14% faster decode step than 3 x 60-bit primes on the integer
    pipe, profiles/r01/params_sweep.md).  Smaller rings keep 60-bit primes."""
    env = os.environ.get("CGB_QBITS")
    if env:
        return int(env)
    return 49 if ring_degree >= 4096 else 60


def ring_for(params, n_limbs: int | None = None, key_seed: int | None = None):
    from .ring import Ring

    log_n, one_row = ring_layout(params.n_slots, params.plain_modulus)
    L = n_limbs or default_limbs(1 << log_n)
    qb = default_qbits(1 << log_n)
    ks = _KEY_SEED if key_seed is None else key_seed
    key = (params.n_slots, params.plain_modulus, L, qb, ks)
    with _rings_lock:
        r = _rings.get(key)
        if r is None:
            seed = np.random.SeedSequence([0xB200_4B45, ks]).generate_state(8, dtype=np.uint32)
            r = Ring(log_n, params.plain_modulus, L, params.n_slots, one_row, seed, q_bits=qb)
            _rings[key] = r
        return r


# ----------------------------------------------------------------------------
# ciphertext storage ownership
# ----------------------------------------------------------------------------
class _Block:
    """Owns a set of arena ids; frees them when the last reference dies."""

    __slots__ = ("ids", "__weakref__")

    def __init__(self, ring, ids: np.ndarray):
        self.ids = ids
        weakref.finalize(self, ring.free, ids)


class GpuCiphertext:
    """Immutable ciphertext handle (replaces SlotCiphertext, backend.py:216-230).

    ``slots`` is a client-side diagnostic: it decrypts on first access with
    the ring's secret key and is read-only, like the reference's array."""

    __slots__ = ("_block", "_aid", "noise_budget", "id", "params", "_ring", "_slots")

    def __init__(self, block: _Block, aid: int, budget: int, cid: int, params, ring):
        self._block, self._aid = block, int(aid)
        self.noise_budget, self.id, self.params, self._ring = int(budget), int(cid), params, ring
        self._slots = None

    def __setattr__(self, name, value):
        if hasattr(self, "_slots") and name != "_slots":
            raise AttributeError("GpuCiphertext is immutable")
        object.__setattr__(self, name, value)

    @property
    def n_slots(self) -> int:
        return self.params.n_slots

    @property
    def slots(self) -> np.ndarray:
        if self._slots is None:
            s = self._ring.decrypt([self._aid])[0]
            s.setflags(write=False)
            object.__setattr__(self, "_slots", s)
        return self._slots

    def words(self) -> np.ndarray:
        """The raw NTT-domain ciphertext words, uint64[2][L][N]."""
        return self._ring.store([self._aid])[0]

    def __repr__(self):
        return f"GpuCiphertext(id={self.id}, budget={self.noise_budget}, slot={self._aid})"


SlotCiphertext = GpuCiphertext


# ----------------------------------------------------------------------------
# waves: batches of ciphertexts processed by one launch sequence
# ----------------------------------------------------------------------------
EXT_B = os.environ.get("CGB_EXT_B", "1") != "0"  # resident base-B extensions of KV cache parts
EXT_A = os.environ.get("CGB_EXT_A", "1") != "0"  # ... and of an a-operand repeated across a mult_cipher wave
_ROT_DEDUP = os.environ.get("CGB_ROT_DEDUP", "1") != "0"  # one key switch per (content class, step)
_ROT_CHAIN = os.environ.get("CGB_ROT_CHAIN", "1") != "0"  # fold / doubling chains as one library call


_class_counter = itertools.count(1)


def _fresh_classes(k: int) -> np.ndarray:
    """k content classes never issued before (positive; wave_of's aid classes are negative)."""
    return np.fromiter((next(_class_counter) for _ in range(k)), dtype=np.int64, count=k)


class Wave:
    """A batch of ciphertexts (arena ids + ledger budgets + owning contexts).

    The fused hot path works on waves so that, e.g., all 64 x 12 broadcast
    chains of a decode step rotate in one batched key switch.  ``owner``
    maps each item to an index into ``ctxs``; counters and ciphertext ids
    (``cids``) are charged to the owning context exactly as the per-op
    path would charge them."""

    __slots__ = ("ctxs", "owner", "aids", "budgets", "blocks", "cids", "klass")

    def __init__(self, ctxs, owner, aids, budgets, blocks, cids=None, klass=None):
        self.ctxs, self.owner, self.aids, self.budgets, self.blocks = ctxs, owner, aids, budgets, blocks
        self.cids = np.zeros(len(aids), np.int64) if cids is None else cids
        # content classes: items with equal klass hold the same ciphertext words
        # (copies of one input, or one rotation of such copies); None = all distinct.
        # w_rotate computes one key switch per (class, step) and copies the rest.
        self.klass = klass

    def __len__(self):
        return int(self.aids.size)

    def take(self, idx) -> "Wave":
        idx = np.asarray(idx, dtype=np.int64).reshape(-1)
        return Wave(self.ctxs, self.owner[idx], self.aids[idx], self.budgets[idx], self.blocks, self.cids[idx],
                    None if self.klass is None else self.klass[idx])

    @staticmethod
    def concat(waves: Sequence["Wave"]) -> "Wave":
        ctxs, owners = [], []
        for w in waves:
            base = len(ctxs)
            ctxs.extend(w.ctxs)
            owners.append(w.owner + base)
        blocks = [b for w in waves for b in w.blocks]
        klass = None
        if any(w.klass is not None for w in waves):
            klass = np.concatenate([w.klass if w.klass is not None else _fresh_classes(len(w)) for w in waves])
        return Wave(ctxs, np.concatenate(owners), np.concatenate([w.aids for w in waves]),
                    np.concatenate([w.budgets for w in waves]), blocks, np.concatenate([w.cids for w in waves]),
                    klass)

    def handles(self) -> list:
        keep = self.blocks[0] if len(self.blocks) == 1 else _Keep(self.blocks)
        out = []
        for i in range(len(self)):
            c = self.ctxs[self.owner[i]]
            out.append(GpuCiphertext(keep, self.aids[i], self.budgets[i], self.cids[i], c.params, c._ring))
        return out


class PlainBatch:
    """A batch of structured plaintext slot vectors named by hashable keys
    (e.g. one-hot masks), so encoded plaintexts are found in the device
    cache without building or hashing the vectors; ``build(keys)`` makes
    the rows only on a cache miss."""

    __slots__ = ("keys", "build")

    def __init__(self, keys, build):
        self.keys, self.build = list(keys), build

    def __len__(self):
        return len(self.keys)


def onehot_batch(n: int, slots) -> PlainBatch:
    slots = [int(j) for j in np.asarray(slots).reshape(-1)]

    def build(ks):
        v = np.zeros((len(ks), n), dtype=np.int64)
        v[np.arange(len(ks)), [k[2] for k in ks]] = 1
        return v

    return PlainBatch([("onehot", n, j) for j in slots], build)


# ----------------------------------------------------------------------------
# the context
# ----------------------------------------------------------------------------
_context_uid = itertools.count()


def residues(values, t: int) -> np.ndarray:
    """int64 residues mod t.  Inputs already in [0, t) (shares, masks, decoded
    slots) are returned as they are: the integer modulo is the costliest host
    pass on the client round trips."""
    arr = np.asarray(values, dtype=np.int64)
    if arr.size == 0 or (arr.min() >= 0 and arr.max() < t):
        return arr
    return np.mod(arr, t)


def _as_slots(values, params) -> np.ndarray:
    arr = np.asarray(values, dtype=np.int64)
    if arr.ndim != 1 or arr.shape[0] != params.n_slots:
        raise ParameterError(f"expected a vector of length {params.n_slots}, got shape {arr.shape}")
    return residues(arr, params.plain_modulus)


class GpuContext:
    """``Context`` (backend.py:245-364) over the B200 RNS-BFV ring."""

    def __init__(self, params, seed=0, n_limbs: int | None = None):
        self.params = params
        self.counter = OpCounter()
        self._seed_seq = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
        self.rng = np.random.default_rng(self._seed_seq)
        self._next_id = next(_context_uid) * 1_000_000_000
        self._ring = ring_for(params, n_limbs)
        ss = self._seed_seq
        self._enc_key = np.random.SeedSequence(ss.entropy, spawn_key=tuple(ss.spawn_key) + (0xB200,)).generate_state(
            8, dtype=np.uint32)
        self._hook_key = np.random.SeedSequence(ss.entropy, spawn_key=tuple(ss.spawn_key) + (0xB201,)).generate_state(
            8, dtype=np.uint32)
        self._enc_index = 0
        self._hook_index = 0
        self._n_limbs = n_limbs

    # -- helpers (backend.py:262-288) ---------------------------------------
    @property
    def ring(self):
        return self._ring

    def plain_vector(self, values) -> PlainVector:
        return _as_slots(values, self.params)

    def plain_from_dense(self, values) -> PlainVector:
        arr = np.asarray(values, dtype=np.int64)
        if arr.shape[0] > self.params.n_slots:
            raise ParameterError("vector longer than slot count")
        out = np.zeros(self.params.n_slots, dtype=np.int64)
        out[: arr.shape[0]] = arr
        return residues(out, self.params.plain_modulus)

    def zeros(self) -> PlainVector:
        return np.zeros(self.params.n_slots, dtype=np.int64)

    def fork(self) -> "GpuContext":
        return GpuContext(self.params, self._seed_seq.spawn(1)[0], self._n_limbs)

    def join(self, child) -> None:
        self.counter.merge(child.counter)

    def _take_ids(self, n: int) -> int:
        base = self._next_id
        self._next_id += n
        return base

    def _new(self, n: int):
        ids = self._ring.alloc(n)
        return _Block(self._ring, ids), ids

    def _check(self, *cts) -> None:
        for ct in cts:
            if not isinstance(ct, GpuCiphertext) or ct.params != self.params:
                raise ParameterError("ciphertext belongs to an incompatible context")

    def _spend(self, budget: int, cost: int) -> int:
        left = budget - cost
        if left < 0:
            raise NoiseBudgetExhausted(f"operation needs {cost} bits but only {budget} remain")
        return left

    def _emit(self, block, aid, budget) -> GpuCiphertext:
        return GpuCiphertext(block, aid, budget, self._take_ids(1), self.params, self._ring)

    # -- plaintext operands ------------------------------------------------------
    def _plaintexts(self, vecs: np.ndarray, kind: int):
        """Encode a batch of slot vectors; returns (owner, ids)."""
        return _pt_cache(self._ring).get(vecs, kind)

    # -- client role ---------------------------------------------------------------
    def _encrypt_slots(self, vecs: np.ndarray, hook: bool = False):
        n = vecs.shape[0]
        blk, ids = self._new(n)
        if hook:
            self._ring.encrypt(vecs, self._hook_key, self._hook_index, ids)
            self._hook_index += n
        else:
            self._ring.encrypt(vecs, self._enc_key, self._enc_index, ids)
            self._enc_index += n
        return blk, ids

    def encrypt(self, v) -> GpuCiphertext:
        slots = _as_slots(v, self.params)
        blk, ids = self._encrypt_slots(slots.reshape(1, -1))
        self.counter.encrypt += 1
        return self._emit(blk, ids[0], self.params.initial_noise_budget)

    def decrypt(self, ct) -> PlainVector:
        self._check(ct)
        if ct.noise_budget <= 0:
            raise DecryptionFailure("noise budget exhausted: decryption would be incorrect")
        self.counter.decrypt += 1
        return self._ring.decrypt([ct._aid])[0]

    # -- server role ---------------------------------------------------------------
    def add(self, a, b) -> GpuCiphertext:
        self._check(a, b)
        budget = self._spend(min(a.noise_budget, b.noise_budget), self.params.noise_costs.add)
        blk, ids = self._new(1)
        self._ring.add([a._aid], [b._aid], ids)
        self.counter.add += 1
        return self._emit(blk, ids[0], budget)

    def add_plain(self, a, v) -> GpuCiphertext:
        self._check(a)
        slots = _as_slots(v, self.params)
        budget = self._spend(a.noise_budget, self.params.noise_costs.add_plain)
        keep, pts = self._plaintexts(slots.reshape(1, -1), nat.CGB_PT_ADD)
        blk, ids = self._new(1)
        self._ring.add_plain([a._aid], pts, ids)
        self.counter.add_plain += 1
        return self._emit(blk, ids[0], budget)

    def mult_plain(self, a, v) -> GpuCiphertext:
        self._check(a)
        slots = _as_slots(v, self.params)
        budget = self._spend(a.noise_budget, self.params.noise_costs.mult_plain)
        keep, pts = self._plaintexts(slots.reshape(1, -1), nat.CGB_PT_MUL)
        blk, ids = self._new(1)
        self._ring.mult_plain([a._aid], pts, ids)
        self.counter.mult_plain += 1
        return self._emit(blk, ids[0], budget)

    def mult_cipher(self, a, b) -> GpuCiphertext:
        self._check(a, b)
        budget = self._spend(min(a.noise_budget, b.noise_budget), self.params.noise_costs.mult_cipher)
        blk, ids = self._new(1)
        self._ring.mult_cipher([a._aid], [b._aid], ids)
        self.counter.mult_cipher += 1
        return self._emit(blk, ids[0], budget)

    def rotate(self, a, k: int) -> GpuCiphertext:
        """Cyclic left shift by k slots (backend.py:349-355)."""
        self._check(a)
        budget = self._spend(a.noise_budget, self.params.noise_costs.rotate)
        blk, ids = self._new(1)
        _rotate_ids(self._ring, self.params, np.array([a._aid], np.uint32), np.array([int(k)], np.int64), ids, False)
        self.counter.rotate += 1
        return self._emit(blk, ids[0], budget)

    def with_budget(self, ct, budget: int):
        """Test hook (backend.py:357-360): same values, explicit budget.

        Raising the ledger above the ciphertext's own budget re-encrypts the
        payload (client role, separate nonce stream, not counted) so that the
        real noise matches the fresh ledger; lowering it is ledger-only."""
        self._check(ct)
        if budget > ct.noise_budget:
            vals = self._ring.decrypt([ct._aid])
            blk, ids = self._encrypt_slots(vals, hook=True)
            return GpuCiphertext(blk, ids[0], budget, ct.id, self.params, self._ring)
        return GpuCiphertext(ct._block, ct._aid, budget, ct.id, self.params, self._ring)

    def load_ciphertext(self, values, budget: int) -> GpuCiphertext:
        """Rehydrate a serialized (decrypted) part; not counted (backend.py:362)."""
        slots = _as_slots(values, self.params)
        blk, ids = self._encrypt_slots(slots.reshape(1, -1), hook=True)
        return self._emit(blk, ids[0], budget)

    def load_ciphertext_words(self, words, budget: int, cid: int | None = None) -> GpuCiphertext:
        """Rehydrate a ciphertext-level snapshot (kv_cache.save_cache_ct): raw
        NTT-domain words uint64[2][L][N] of this context's ring, loaded without
        decryption; not counted.  ``cid`` restores the snapshot's ciphertext id
        (the same ciphertext), else a fresh id is issued as load_ciphertext does
        (backend.py:362-364)."""
        r = self._ring
        w = np.ascontiguousarray(np.asarray(words, dtype=np.uint64))
        if w.shape != (2, r.L, r.N):
            raise ParameterError(f"ciphertext words of shape {w.shape}, this ring needs {(2, r.L, r.N)}")
        mods = np.asarray(r.moduli[: r.L], dtype=np.uint64).reshape(1, r.L, 1)
        if (w >= mods).any():
            raise ParameterError("ciphertext words are not residues of this ring's moduli")
        blk, ids = self._new(1)
        r.load(ids, w.reshape(1, 2, r.L, r.N))
        if cid is None:
            return self._emit(blk, ids[0], budget)
        return GpuCiphertext(blk, ids[0], budget, int(cid), self.params, r)

    # -- diagnostics -------------------------------------------------------------------
    def noise_budget_bits(self, ct) -> float:
        """Real invariant noise budget (bits) of a ciphertext; client-side."""
        return float(self._ring.noise_budget([ct._aid])[0])

    # =============================================================================
    # wave API (batched; used by the fused hot path)
    # =============================================================================
    @staticmethod
    def wave_of(cts: Sequence[GpuCiphertext], ctxs=None) -> Wave:
        cts = list(cts)
        if ctxs is None:
            ctxs = [None]
            owner = np.zeros(len(cts), dtype=np.int64)
        else:
            ctxs, owner = _owners(ctxs)
        aids = np.array([c._aid for c in cts], dtype=np.uint32)
        budgets = np.array([c.noise_budget for c in cts], dtype=np.int64)
        cids = np.array([c.id for c in cts], dtype=np.int64)
        # one live arena id is one ciphertext: repeated handles share a content class
        klass = -(aids.astype(np.int64) + 1) if len(set(aids.tolist())) < len(aids) else None
        return Wave(ctxs, owner, aids, budgets, [c._block for c in cts], cids, klass)

    @staticmethod
    def bind(wave: Wave, ctx) -> Wave:
        return Wave([ctx], np.zeros(len(wave), np.int64), wave.aids, wave.budgets, wave.blocks, wave.cids, wave.klass)

    # -- wave primitives: each charges counters/ids to the owning contexts exactly
    # -- as the equivalent sequence of per-op calls would
    @staticmethod
    def _charge(wave: Wave, field_name: str, n_emit: int = 1, counts=None) -> np.ndarray:
        """Bump the owners' counters; returns the ids the emitted items get
        (item order within each owner, n_emit ids per item, last one kept)."""
        counts = np.bincount(wave.owner, minlength=len(wave.ctxs)) if counts is None else counts
        for c, k in zip(wave.ctxs, counts):
            if k:
                setattr(c.counter, field_name, getattr(c.counter, field_name) + int(k))
        if n_emit == 0:
            return wave.cids
        cids = np.empty(len(wave), np.int64)
        for o, c in enumerate(wave.ctxs):
            sel = np.nonzero(wave.owner == o)[0]
            if sel.size:
                cids[sel] = c._next_id + n_emit * np.arange(sel.size) + (n_emit - 1)
                c._next_id += n_emit * sel.size
        return cids

    @staticmethod
    def _spend_all(budgets: np.ndarray, cost: int) -> np.ndarray:
        left = budgets - cost
        if left.size and left.min() < 0:
            i = int(np.argmin(left))
            raise NoiseBudgetExhausted(f"operation needs {cost} bits but only {int(budgets[i])} remain")
        return left

    @staticmethod
    def _derive(wave: Wave, aids, budgets, block) -> Wave:
        return Wave(wave.ctxs, wave.owner, aids, budgets, [block])

    @staticmethod
    def w_encrypt(ctxs, vecs, canonical: bool = False) -> Wave:
        """Encrypt rows of ``vecs`` (item i by ctxs[i]); one nonce per item in order.
        ``canonical``: the rows are residues in [0, t) by construction (shares,
        decrypted slots), so the host range passes are skipped."""
        uniq, owner = _owners(ctxs)
        vecs = np.ascontiguousarray(vecs if canonical else residues(vecs, uniq[0].params.plain_modulus))
        ring = uniq[0]._ring
        ids = ring.alloc(len(owner))
        blk = _Block(ring, ids)
        # item i takes its context's next encryption index, in item order (the per-context
        # sequence of Context.encrypt calls); all contexts go through one launch sequence
        idx = np.zeros(len(owner), np.uint64)
        for k, c in enumerate(uniq):
            sel = np.nonzero(owner == k)[0]
            idx[sel] = c._enc_index + np.arange(sel.size, dtype=np.uint64)
            c._enc_index += sel.size
        keys = np.stack([np.asarray(c._enc_key, dtype=np.uint32).reshape(8) for c in uniq])[owner]
        ring.encrypt_batch(vecs, keys, idx, ids, canonical=True)
        w = Wave(uniq, owner, ids, np.full(len(owner), uniq[0].params.initial_noise_budget, np.int64), [blk])
        w.cids = GpuContext._charge(w, "encrypt")
        return w

    @staticmethod
    def w_reencrypt(wave: Wave, ctxs) -> Wave:
        """w_encrypt(ctxs, w_decrypt(wave)) -- the client's re-encryption of a refresh
        (kv_cache.py:150) -- with the slot vectors kept on the device: the same
        words, counters, nonces and budgets as the two calls."""
        if len(wave) and wave.budgets.min() <= 0:
            raise DecryptionFailure("noise budget exhausted: decryption would be incorrect")
        GpuContext._charge(wave, "decrypt", n_emit=0)
        uniq, owner = _owners(ctxs)
        ring = uniq[0]._ring
        ids = ring.alloc(len(owner))
        blk = _Block(ring, ids)
        idx = np.zeros(len(owner), np.uint64)
        for k, c in enumerate(uniq):
            sel = np.nonzero(owner == k)[0]
            idx[sel] = c._enc_index + np.arange(sel.size, dtype=np.uint64)
            c._enc_index += sel.size
        keys = np.stack([np.asarray(c._enc_key, dtype=np.uint32).reshape(8) for c in uniq])[owner]
        ring.reencrypt_batch(wave.aids, keys, idx, ids)
        w = Wave(uniq, owner, ids, np.full(len(owner), uniq[0].params.initial_noise_budget, np.int64), [blk])
        w.cids = GpuContext._charge(w, "encrypt")
        return w

    @staticmethod
    def w_decrypt(wave: Wave) -> np.ndarray:
        if len(wave) == 0:
            return np.zeros((0, wave.ctxs[0].params.n_slots), np.int64)
        if wave.budgets.min() <= 0:
            raise DecryptionFailure("noise budget exhausted: decryption would be incorrect")
        GpuContext._charge(wave, "decrypt", n_emit=0)
        return wave.ctxs[0]._ring.decrypt(wave.aids)

    @staticmethod
    def w_decrypt_start(wave: Wave):
        """w_decrypt split at the client round trip: charges and enqueues now;
        w_decrypt_finish(pending) waits for this batch only."""
        if len(wave) == 0:
            return ("empty", wave.ctxs[0].params.n_slots)
        if wave.budgets.min() <= 0:
            raise DecryptionFailure("noise budget exhausted: decryption would be incorrect")
        GpuContext._charge(wave, "decrypt", n_emit=0)
        ring = wave.ctxs[0]._ring
        return (ring, ring.decrypt_start(wave.aids), wave)

    @staticmethod
    def w_decrypt_finish(pending) -> np.ndarray:
        if pending[0] == "empty":
            return np.zeros((0, pending[1]), np.int64)
        ring, ticket, _ = pending
        return ring.decrypt_finish(ticket)

    @staticmethod
    def w_add(wa: Wave, wb: Wave) -> Wave:
        c0 = wa.ctxs[0]
        b = GpuContext._spend_all(np.minimum(wa.budgets, wb.budgets), c0.params.noise_costs.add)
        blk, ids = c0._new(len(wa))
        c0._ring.add(wa.aids, wb.aids, ids)
        return Wave(wa.ctxs, wa.owner, ids, b, [blk], GpuContext._charge(wa, "add"))

    @staticmethod
    def _plain_op(wave: Wave, vecs, kind, field_name, one_shot: bool = False, canonical: bool = False):
        c0 = wave.ctxs[0]
        cost = getattr(c0.params.noise_costs, field_name)
        b = GpuContext._spend_all(wave.budgets, cost)
        if not isinstance(vecs, PlainBatch):
            vecs = np.asarray(vecs, dtype=np.int64) if canonical else residues(vecs, c0.params.plain_modulus)
            if vecs.ndim == 1:
                vecs = np.broadcast_to(vecs, (len(wave), vecs.shape[0]))
        ring = c0._ring
        fn = ring.add_plain if kind == nat.CGB_PT_ADD else ring.mult_plain
        blk, ids = c0._new(len(wave))
        if one_shot and not isinstance(vecs, PlainBatch):
            # random masks never recur: encode into scratch plaintexts, no hashing, no cache
            _pt_cache(ring).make_room(len(wave))
            pts = ring.alloc_pt(len(wave))
            try:
                ring.encode_pt(vecs, kind, pts, canonical=True)
                fn(wave.aids, pts, ids)
            finally:
                ring.free_pt(pts)  # stream-ordered: later encodes run after this op
        else:
            _, pts = c0._plaintexts(vecs, kind)
            fn(wave.aids, pts, ids)
        return Wave(wave.ctxs, wave.owner, ids, b, [blk], GpuContext._charge(wave, field_name))

    @staticmethod
    def w_add_plain(wave: Wave, vecs, one_shot: bool = False, canonical: bool = False) -> Wave:
        return GpuContext._plain_op(wave, vecs, nat.CGB_PT_ADD, "add_plain", one_shot, canonical)

    @staticmethod
    def w_add_plain_ids(wave: Wave, pts) -> Wave:
        """add_plain per item with already-encoded plaintexts (arena ids of kind
        CGB_PT_ADD, e.g. device-drawn masks); charged like w_add_plain."""
        c0 = wave.ctxs[0]
        b = GpuContext._spend_all(wave.budgets, c0.params.noise_costs.add_plain)
        blk, ids = c0._new(len(wave))
        c0._ring.add_plain(wave.aids, pts, ids)
        return Wave(wave.ctxs, wave.owner, ids, b, [blk], GpuContext._charge(wave, "add_plain"))

    @staticmethod
    def w_mult_plain(wave: Wave, vecs, one_shot: bool = False) -> Wave:
        return GpuContext._plain_op(wave, vecs, nat.CGB_PT_MUL, "mult_plain", one_shot)

    @staticmethod
    def w_mult_cipher(wa: Wave, wb: Wave, resident_b: bool = False) -> Wave:
        """mult_cipher per item; ``resident_b``: wb's items are multiplied again
        later (KV cache parts), so their base-B extension is computed once and kept
        with the ciphertext (same words either way)."""
        c0 = wa.ctxs[0]
        b = GpuContext._spend_all(np.minimum(wa.budgets, wb.budgets), c0.params.noise_costs.mult_cipher)
        blk, ids = c0._new(len(wa))
        ring = c0._ring
        if resident_b and EXT_B:
            bx = ring.ext_B(wb.aids)
            if EXT_A and (ring.has_ext(wa.aids) or (len(wa) >= 8 and 4 * np.unique(wa.aids).size <= len(wa))):
                # a repeats (one ciphertext times many), or already has a resident extension
                # (a sweep's operand extended once for all its waves): no per-item extension
                ring.mult_cipher_ext2(wa.aids, ring.ext_B(wa.aids), wb.aids, bx, ids)
            else:
                ring.mult_cipher_ext(wa.aids, wb.aids, bx, ids)
        else:
            ring.mult_cipher(wa.aids, wb.aids, ids)
        return Wave(wa.ctxs, wa.owner, ids, b, [blk], GpuContext._charge(wa, "mult_cipher"))

    @staticmethod
    def w_rotate(wave: Wave, steps, add_input: bool = False) -> Wave:
        """rotate(a, k) per item; with add_input, add(a, rotate(a, k)) (the
        doubling / folding step), fused into the key-switch epilogue."""
        c0 = wave.ctxs[0]
        costs = c0.params.noise_costs
        st = np.ascontiguousarray(np.broadcast_to(np.asarray(steps, dtype=np.int64), (len(wave),)))
        rb = GpuContext._spend_all(wave.budgets, costs.rotate)
        b = GpuContext._spend_all(np.minimum(wave.budgets, rb), costs.add) if add_input else rb
        klass = None
        if wave.klass is not None and _ROT_DEDUP:
            # one key switch per distinct (content class, step); the other items share
            # its arena id -- the same words their own key switch would give (handles
            # are immutable and the block frees each id once)
            _, fi, inv = np.unique(np.stack([wave.klass, st], axis=1), axis=0, return_index=True,
                                   return_inverse=True)
            lead = fi[inv.reshape(-1)].astype(np.int64)  # first item of each (class, step)
            first = np.flatnonzero(lead == np.arange(len(wave)))
            blk, uids = c0._new(first.size)
            _rotate_ids(c0._ring, c0.params, wave.aids[first], st[first], uids, add_input)
            ids = np.empty(len(wave), np.uint32)
            ids[first] = uids
            dup = np.flatnonzero(lead != np.arange(len(wave)))
            ids[dup] = ids[lead[dup]]
            fresh = _fresh_classes(first.size)
            cls = np.empty(len(wave), np.int64)
            cls[first] = fresh
            cls[dup] = cls[lead[dup]]
            klass = cls if dup.size else None
        else:
            blk, ids = c0._new(len(wave))
            _rotate_ids(c0._ring, c0.params, wave.aids, st, ids, add_input)
        if add_input:
            GpuContext._charge(wave, "rotate", n_emit=0)
            cids = GpuContext._charge(wave, "add", n_emit=2)
        else:
            cids = GpuContext._charge(wave, "rotate")
        return Wave(wave.ctxs, wave.owner, ids, b, [blk], cids, klass)

    @staticmethod
    def w_rotate_add_chain(wave: Wave, steps) -> Wave:
        """``wave <- w_rotate(wave, s, add_input=True)`` for s in steps, as ONE library
        call (cgb_rotate_add_chain): the same words, budgets, counters and ciphertext
        ids as the loop -- the intermediate ciphertexts never get arena slots and the
        per-wave host work is paid once (small fold waves are host-bound).  Falls back
        to the loop whenever the closed forms below would not describe it: repeated
        handles (content classes), the two-row layout, a step that is a multiple of
        the slot count, or a budget the chain would exhaust (the loop then raises at
        the exact step)."""
        steps = [int(s) for s in steps]
        if not steps:
            return wave
        c0 = wave.ctxs[0]
        costs = c0.params.noise_costs
        per = costs.rotate + costs.add
        n = c0.params.n_slots
        if (not _ROT_CHAIN or len(steps) < 2 or wave.klass is not None or not c0._ring.one_row
                or any(s % n == 0 for s in steps)
                or (len(wave) and int(wave.budgets.min()) - per * len(steps) < 0)):
            for s in steps:
                wave = GpuContext.w_rotate(wave, s, add_input=True)
            return wave
        K = len(steps)
        blk, ids = c0._new(len(wave))
        c0._ring.rotate_add_chain(wave.aids, steps, ids)
        # K rotates and K adds per item; each step emits two ids per item (the rotation's,
        # then the sum's, which the item keeps), item order within each owner
        counts = np.bincount(wave.owner, minlength=len(wave.ctxs))
        cids = np.empty(len(wave), np.int64)
        for o, c in enumerate(wave.ctxs):
            k = int(counts[o])
            if not k:
                continue
            c.counter.rotate += K * k
            c.counter.add += K * k
            sel = np.nonzero(wave.owner == o)[0]
            cids[sel] = c._next_id + (K - 1) * 2 * k + 2 * np.arange(k) + 1
            c._next_id += K * 2 * k
        return Wave(wave.ctxs, wave.owner, ids, wave.budgets - per * K, [blk], cids)

    @staticmethod
    def w_sum(wave: Wave, groups) -> Wave:
        """Left-fold sum of each index group (len-1 adds per group, exact mod q
        so one batched reduction gives the sequential fold's words)."""
        c0 = wave.ctxs[0]
        cost = c0.params.noise_costs.add
        groups = [np.asarray(g, dtype=np.int64) for g in groups]
        blk, ids = c0._new(len(groups))
        budgets = np.empty(len(groups), np.int64)
        owner = np.empty(len(groups), np.int64)
        cids = np.empty(len(groups), np.int64)
        for gi, g in enumerate(groups):
            if g.size == 0:
                raise ParameterError("empty sum")
            # the left fold acc <- min(acc, b_t) - cost in closed form: the final budget is
            # min(b_0 - m cost, b_t - (m - t + 1) cost); the sequence strictly decreases,
            # so only the final value can signal exhaustion (the loop then names the step)
            bg = wave.budgets[g]
            m = g.size - 1
            coef = m + 1 - np.arange(g.size)
            coef[0] = m
            acc = int(np.min(bg - coef * cost))
            if acc < 0:
                acc = int(bg[0])
                for b in bg[1:]:
                    acc = min(acc, int(b)) - cost
                    if acc < 0:
                        raise NoiseBudgetExhausted(f"operation needs {cost} bits but only {acc + cost} remain")
            budgets[gi] = acc
            o = owner[gi] = wave.owner[g[0]]
            c = wave.ctxs[o]
            if g.size == 1:
                c0._ring.copy(wave.aids[g], ids[gi:gi + 1])
                cids[gi] = wave.cids[g[0]]
            else:
                c0._ring.sum(wave.aids[g], int(ids[gi]))
                c.counter.add += int(g.size - 1)
                c._next_id += int(g.size - 1)
                cids[gi] = c._next_id - 1
        return Wave(wave.ctxs, owner, ids, budgets, [blk], cids)


class _Keep:
    """Keeps a list of blocks alive for a handle carved from a wave."""

    __slots__ = ("blocks",)

    def __init__(self, blocks):
        self.blocks = blocks


def _owners(ctxs):
    uniq, owner, seen = [], [], {}
    for c in ctxs:
        k = id(c)
        if k not in seen:
            seen[k] = len(uniq)
            uniq.append(c)
        owner.append(seen[k])
    return uniq, np.asarray(owner, dtype=np.int64)


Context = GpuContext


def new_context(params, seed=0) -> GpuContext:
    """backend.py:367-368 -- always the GPU context; fails loudly without CUDA."""
    return GpuContext(params, seed)


# ----------------------------------------------------------------------------
# rotation (one-row native, two-row composed)
# ----------------------------------------------------------------------------
def _rotate_ids(ring, params, a: np.ndarray, steps: np.ndarray, out: np.ndarray, add_input: bool):
    if ring.one_row:
        ring.rotate(a, steps, out, add_input=add_input)
        return
    n = params.n_slots
    h = n // 2
    two_n = 2 * ring.N
    cnt = a.size
    ga = ring.alloc(cnt)
    gb = ring.alloc(cnt)
    try:
        kk = np.mod(steps, n)
        g_plain = np.empty(cnt, np.uint64)
        g_swap = np.empty(cnt, np.uint64)
        masks = np.zeros((cnt, n), dtype=np.int64)
        col = np.arange(n) % h
        for i, k in enumerate(kk):
            kr = int(k) % h
            e = pow(5, kr, two_n)
            g_plain[i], g_swap[i] = e, two_n - e
            keep = col < h - kr
            # k < h: plain rotation where the column does not wrap, row swap where it does
            masks[i] = keep if k < h else ~keep
        ring.galois(a, g_plain, ga)
        ring.galois(a, g_swap, gb)
        cache = _pt_cache(ring)
        kp, pm = cache.get(masks, nat.CGB_PT_MUL)
        kq, pq = cache.get(1 - masks, nat.CGB_PT_MUL)
        ring.mult_plain(ga, pm, ga)
        ring.mult_plain(gb, pq, gb)
        if add_input:
            ring.add(ga, gb, gb)
            ring.add(gb, a, out)
        else:
            ring.add(ga, gb, out)
    finally:
        ring.free(ga)
        ring.free(gb)


# ----------------------------------------------------------------------------
# device plaintext cache (content-addressed)
# ----------------------------------------------------------------------------
class _PtCache:
    """Content-hashed cache of encoded plaintexts (one-hot masks, append masks
    and block masks recur every step).  Entries are evicted LRU."""

    def __init__(self, ring, capacity: int):
        self.ring, self.capacity = ring, capacity
        self.map: dict = {}
        self.lock = threading.Lock()
        self.tick = 0

    def get(self, vecs, kind: int):
        if isinstance(vecs, PlainBatch):
            keys = [(kind,) + tuple(k) for k in vecs.keys]
            build = vecs.build
        else:
            vecs = np.ascontiguousarray(np.asarray(vecs, dtype=np.int64))
            keys = [(kind, hashlib.blake2b(row.tobytes(), digest_size=16).digest()) for row in vecs]
            build = None
        n = len(keys)
        out = np.empty(n, dtype=np.uint32)
        with self.lock:
            missing = []
            for i, k in enumerate(keys):
                ent = self.map.get(k)
                if ent is None:
                    missing.append(i)
                else:
                    self.tick += 1
                    ent[1] = self.tick
                    out[i] = ent[0]
            if missing:
                uniq = {}
                for i in missing:
                    uniq.setdefault(keys[i], []).append(i)
                self._evict(len(uniq))
                ids = self.ring.alloc_pt(len(uniq))
                if build is not None:
                    rows = build([k[1:] for k in uniq])
                else:
                    rows = np.stack([vecs[v[0]] for v in uniq.values()])
                self.ring.encode_pt(rows, kind, ids)
                for pid, (k, idxs) in zip(ids, uniq.items()):
                    self.tick += 1
                    self.map[k] = [int(pid), self.tick]
                    out[idxs] = pid
        return None, out

    def make_room(self, need: int):
        """Leave `need` arena slots free for scratch (one-shot) plaintexts."""
        with self.lock:
            self._evict(need)

    def _evict(self, need: int):
        free = self.ring.arena_pts - len(self.map)
        if free >= need:
            return
        victims = sorted(self.map.items(), key=lambda kv: kv[1][1])[: need - free + 64]
        # pending launches may still read these plaintexts: order after them
        self.ring.sync()
        self.ring.free_pt([v[1][0] for v in victims])
        for k, _ in victims:
            del self.map[k]


_pt_caches: dict = {}


def _pt_cache(ring) -> _PtCache:
    c = _pt_caches.get(id(ring))
    if c is None or c.ring is not ring:
        c = _PtCache(ring, ring.arena_pts)
        _pt_caches[id(ring)] = c
    return c
