"""ctypes wrapper over oracle/rnsbfv.c -- the CPU RNS-BFV restatement.

TEST INFRASTRUCTURE ONLY (the checker): imported by tests/, by
``__graft_entry__.smoke()`` and by bench.py's cpu_baseline leg, never by the
product package.  See the header of rnsbfv.c for what it restates and for
its parity status (polynomial level unpinned against the reference, slot
level pinned through tests/golden/).

Ciphertext layout (shared with the GPU library, include/cgb200.h):
``uint64[2][L][N]`` -- poly (c0, c1), RNS limb over Q, NTT-domain word.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "build" / "librnsbfv_oracle.so"

_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


def build() -> Path:
    """Compile the oracle with its Makefile (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists() or _SO.stat().st_mtime < (_HERE / "rnsbfv.c").stat().st_mtime:
            build()
        L = ctypes.CDLL(str(_SO))
        L.ora_create.restype = ctypes.c_void_p
        L.ora_create.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _u32p,
                                 ctypes.c_int]
        L.ora_destroy.argtypes = [ctypes.c_void_p]
        L.ora_moduli.argtypes = [ctypes.c_void_p, _u64p]
        L.ora_moduli.restype = ctypes.c_int
        L.ora_secret.argtypes = [ctypes.c_void_p, _i64p]
        for name in ("ora_ntt", "ora_intt"):
            getattr(L, name).argtypes = [ctypes.c_void_p, ctypes.c_int, _u64p]
        for name in ("ora_ntt_t", "ora_intt_t"):
            getattr(L, name).argtypes = [ctypes.c_void_p, _u64p]
        L.ora_encode.argtypes = [ctypes.c_void_p, _u64p, _u64p]
        L.ora_decode.argtypes = [ctypes.c_void_p, _u64p, _u64p]
        L.ora_encrypt.argtypes = [ctypes.c_void_p, _u64p, _u32p, ctypes.c_uint64, _u64p]
        L.ora_decrypt.argtypes = [ctypes.c_void_p, _u64p, _u64p]
        L.ora_add.argtypes = [ctypes.c_void_p, _u64p, _u64p, _u64p]
        L.ora_add_plain.argtypes = [ctypes.c_void_p, _u64p, _u64p, _u64p]
        L.ora_mult_plain.argtypes = [ctypes.c_void_p, _u64p, _u64p, _u64p]
        L.ora_mult_cipher.argtypes = [ctypes.c_void_p, _u64p, _u64p, _u64p]
        L.ora_galois.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_uint64, _u64p]
        L.ora_noise_budget.argtypes = [ctypes.c_void_p, _u64p]
        L.ora_noise_budget.restype = ctypes.c_double
        _lib = L
    return _lib


class OracleRing:
    """One parameter set of the restatement (ring, primes, keys)."""

    def __init__(self, log_n: int, t: int, n_limbs: int, n_slots: int, one_row: bool, keyseed, q_bits: int = 60):
        self.log_n, self.N, self.t, self.L = log_n, 1 << log_n, int(t), n_limbs
        self.n_slots, self.one_row = n_slots, bool(one_row)
        ks = np.ascontiguousarray(np.asarray(keyseed, dtype=np.uint32))
        assert ks.shape == (8,)
        self._h = lib().ora_create(log_n, self.t, n_limbs, n_slots, int(one_row), ks, int(q_bits))
        mods = np.zeros(64, dtype=np.uint64)
        k = lib().ora_moduli(self._h, mods)
        self.moduli = [int(x) for x in mods[:k]]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.ora_destroy(h)
            self._h = None

    # shapes -------------------------------------------------------------
    def ct_shape(self):
        return (2, self.L, self.N)

    def new_ct(self):
        return np.zeros(self.ct_shape(), dtype=np.uint64)

    # primitives ---------------------------------------------------------
    def secret(self) -> np.ndarray:
        s = np.zeros(self.N, dtype=np.int64)
        lib().ora_secret(self._h, s)
        return s

    def ntt(self, mod_index: int, a) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().ora_ntt(self._h, mod_index, a)
        return a

    def intt(self, mod_index: int, a) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().ora_intt(self._h, mod_index, a)
        return a

    def ntt_t(self, a) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().ora_ntt_t(self._h, a)
        return a

    def encode(self, slots) -> np.ndarray:
        s = np.ascontiguousarray(np.mod(np.asarray(slots, dtype=np.int64), self.t).astype(np.uint64))
        m = np.zeros(self.N, dtype=np.uint64)
        lib().ora_encode(self._h, s, m)
        return m

    def decode(self, m) -> np.ndarray:
        out = np.zeros(self.n_slots, dtype=np.uint64)
        lib().ora_decode(self._h, np.ascontiguousarray(m, dtype=np.uint64), out)
        return out.astype(np.int64)

    def encrypt_poly(self, m, enc_key, index: int) -> np.ndarray:
        ct = self.new_ct()
        k = np.ascontiguousarray(np.asarray(enc_key, dtype=np.uint32))
        lib().ora_encrypt(self._h, np.ascontiguousarray(m, dtype=np.uint64), k, int(index), ct)
        return ct

    def encrypt(self, slots, enc_key, index: int) -> np.ndarray:
        return self.encrypt_poly(self.encode(slots), enc_key, index)

    def decrypt_poly(self, ct) -> np.ndarray:
        m = np.zeros(self.N, dtype=np.uint64)
        lib().ora_decrypt(self._h, np.ascontiguousarray(ct, dtype=np.uint64), m)
        return m

    def decrypt(self, ct) -> np.ndarray:
        return self.decode(self.decrypt_poly(ct))

    def _binary(self, fn, a, b):
        out = self.new_ct()
        fn(self._h, np.ascontiguousarray(a, dtype=np.uint64), np.ascontiguousarray(b, dtype=np.uint64), out)
        return out

    def add(self, a, b):
        return self._binary(lib().ora_add, a, b)

    def add_plain(self, a, slots):
        return self._binary(lib().ora_add_plain, a, self.encode(slots))

    def mult_plain(self, a, slots):
        return self._binary(lib().ora_mult_plain, a, self.encode(slots))

    def mult_cipher(self, a, b):
        return self._binary(lib().ora_mult_cipher, a, b)

    def galois(self, a, g: int):
        out = self.new_ct()
        lib().ora_galois(self._h, np.ascontiguousarray(a, dtype=np.uint64), int(g), out)
        return out

    def galois_elt(self, k: int) -> int:
        """Galois element of a cyclic left shift by k (one-row layout)."""
        assert self.one_row
        return pow(5, k % self.n_slots, 2 * self.N)

    def rotate(self, a, k: int):
        return self.galois(a, self.galois_elt(k))

    def noise_budget(self, ct) -> float:
        return lib().ora_noise_budget(self._h, np.ascontiguousarray(ct, dtype=np.uint64))
