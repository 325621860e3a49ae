"""Per-op ``Context`` over the CPU RNS-BFV oracle (oracle/rnsbfv.c).

TEST INFRASTRUCTURE ONLY (the checker).  Restates the method set of the
reference's substrate ``cryptogen.backend.Context`` (/root/reference/pkg/
src/cryptogen/backend.py:262-364: encrypt :307, decrypt :312, add :321,
add_plain :327, mult_plain :334, mult_cipher :341, rotate :349, the ledger
``_spend`` :295-301 and the op counters :173-213) with real RNS-BFV
ciphertexts computed by ``OracleRing``, one scalar C call per op.

Running the reference's per-op hot path (oracle/reference_path.py, which
follows arcc.py:320-379 and kv_cache.py:114-196 op by op) over this context
gives the ciphertext words the reference's op sequence produces under the
RNS-BFV restatement; tests/test_gpu_ring_parity.py compares them with the
B200 wave schedule word for word.  Encryption randomness follows the GPU
context's convention (ChaCha20 keyed by the context's ``_enc_key``, one
nonce index per encryption in call order), so a context built from a
``GpuContext``'s key and next index reproduces its encryptions.
"""

from __future__ import annotations

import itertools

import numpy as np

from paper_2602_08798_b200.backend import DecryptionFailure, NoiseBudgetExhausted, OpCounter, ParameterError

_uid = itertools.count(1)


class OracleCt:
    """Immutable ciphertext handle: words uint64[2][L][N] + ledger budget + id."""

    __slots__ = ("w", "noise_budget", "id", "params")

    def __init__(self, w, budget, cid, params):
        w = np.ascontiguousarray(w, dtype=np.uint64)
        w.setflags(write=False)
        self.w, self.noise_budget, self.id, self.params = w, int(budget), int(cid), params

    def words(self) -> np.ndarray:
        return self.w


class OracleContext:
    def __init__(self, params, ring, enc_key, enc_index: int = 0):
        self.params, self.ring = params, ring
        self.counter = OpCounter()
        self._enc_key = np.ascontiguousarray(np.asarray(enc_key, dtype=np.uint32).reshape(8))
        self._enc_index = int(enc_index)

    # helpers (backend.py:262-288)
    def _slots(self, v):
        a = np.asarray(v, dtype=np.int64)
        if a.ndim != 1 or a.shape[0] != self.params.n_slots:
            raise ParameterError(f"expected a vector of length {self.params.n_slots}, got shape {a.shape}")
        return np.mod(a, self.params.plain_modulus)

    def plain_vector(self, v):
        return self._slots(v)

    def plain_from_dense(self, v):
        a = np.asarray(v, dtype=np.int64)
        out = np.zeros(self.params.n_slots, dtype=np.int64)
        out[: a.shape[0]] = a
        return np.mod(out, self.params.plain_modulus)

    def zeros(self):
        return np.zeros(self.params.n_slots, dtype=np.int64)

    def _spend(self, budget, cost):
        left = budget - cost
        if left < 0:
            raise NoiseBudgetExhausted(f"operation needs {cost} bits but only {budget} remain")
        return left

    def _emit(self, w, budget):
        return OracleCt(w, budget, next(_uid), self.params)

    def wrap(self, words, budget) -> OracleCt:
        """A handle over existing ciphertext words (e.g. a GPU cache part)."""
        return self._emit(words, budget)

    # client role
    def encrypt(self, v):
        w = self.ring.encrypt(self._slots(v), self._enc_key, self._enc_index)
        self._enc_index += 1
        self.counter.encrypt += 1
        return self._emit(w, self.params.initial_noise_budget)

    def decrypt(self, ct):
        if ct.noise_budget <= 0:
            raise DecryptionFailure("noise budget exhausted: decryption would be incorrect")
        self.counter.decrypt += 1
        return self.ring.decrypt(ct.w)

    # server role
    def add(self, a, b):
        self.counter.add += 1
        return self._emit(self.ring.add(a.w, b.w),
                          self._spend(min(a.noise_budget, b.noise_budget), self.params.noise_costs.add))

    def add_plain(self, a, v):
        self.counter.add_plain += 1
        return self._emit(self.ring.add_plain(a.w, self._slots(v)),
                          self._spend(a.noise_budget, self.params.noise_costs.add_plain))

    def mult_plain(self, a, v):
        self.counter.mult_plain += 1
        return self._emit(self.ring.mult_plain(a.w, self._slots(v)),
                          self._spend(a.noise_budget, self.params.noise_costs.mult_plain))

    def mult_cipher(self, a, b):
        self.counter.mult_cipher += 1
        return self._emit(self.ring.mult_cipher(a.w, b.w),
                          self._spend(min(a.noise_budget, b.noise_budget), self.params.noise_costs.mult_cipher))

    def rotate(self, a, k: int):
        self.counter.rotate += 1
        return self._emit(self.ring.rotate(a.w, int(k)), self._spend(a.noise_budget, self.params.noise_costs.rotate))
