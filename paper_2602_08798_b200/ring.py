"""Thin host object over one ``cgb_ring`` (include/cgb200.h).

A ring is the device-side realisation of one ``BackendParams`` value: the
ring degree, the prime chains, the secret key, the evaluation keys and the
ciphertext/plaintext arenas.  Ciphertexts and plaintexts are named by
uint32 arena ids; every method is batched over arrays of ids.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native as nat

DEFAULT_ARENA_BYTES = int(os.environ.get("CGB_ARENA_GIB", "24")) << 30
DEFAULT_PT_BYTES = int(os.environ.get("CGB_PT_ARENA_GIB", "4")) << 30


def _ids(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32).reshape(-1))


class Ring:
    def __init__(self, log_n: int, t: int, n_limbs: int, n_slots: int, one_row: bool, key_seed,
                 arena_cts: int | None = None, arena_pts: int | None = None, q_bits: int = 60):
        self.log_n, self.N, self.t, self.L = log_n, 1 << log_n, int(t), int(n_limbs)
        self.n_slots, self.one_row = int(n_slots), bool(one_row)
        self.q_bits = int(q_bits)
        # the library's NTT pipe (build_ring): FP64 for rings of primes < 2^49 from 2^12 up
        self.fp_ntt = log_n >= 12 and self.q_bits <= 49 and not os.environ.get("CGB_INT_NTT")
        self.ct_words = 2 * self.L * self.N
        if arena_cts is None:
            arena_cts = max(64, min(1 << 20, DEFAULT_ARENA_BYTES // (8 * self.ct_words)))
        if arena_pts is None:
            arena_pts = max(64, min(1 << 20, DEFAULT_PT_BYTES // (8 * self.L * self.N)))
        self.arena_cts, self.arena_pts = int(arena_cts), int(arena_pts)
        self._ext = {}  # arena id -> the two slots of its resident base-B extension (cgb_extend_b)
        self.h2d_bytes = 0  # host payload bytes moved to / from the device (slot vectors, raw words)
        self.d2h_bytes = 0
        ks = np.ascontiguousarray(np.asarray(key_seed, dtype=np.uint32).reshape(8))
        h = ctypes.c_void_p()
        L = nat.lib()
        nat.check(L.cgb_ring_create_ex(log_n, self.t, self.L, int(q_bits), self.n_slots, int(one_row), nat.u32ptr(ks),
                                       self.arena_cts, self.arena_pts, ctypes.byref(h)), "cgb_ring_create")
        self._h = h
        mods = np.zeros(64, dtype=np.uint64)
        k = L.cgb_ring_moduli(self._h, nat.u64ptr(mods), 64)
        self.moduli = [int(x) for x in mods[:k]]

    def close(self):
        if getattr(self, "_h", None):
            nat.lib().cgb_ring_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------
    @property
    def handle(self):
        return self._h

    def launches(self) -> int:
        return int(nat.lib().cgb_launch_count(self._h))

    def timing(self, on: int):
        """0 off, 1 every launch (PDL off), 2 every multi-launch operation as one record."""
        nat.check(nat.lib().cgb_timing_enable(self._h, int(on)), "cgb_timing_enable")

    def timing_report(self) -> dict:
        """{kernel: (launches, total_ms, algorithmic_bytes, algorithmic_modmuls)} of the recorded launches."""
        buf = ctypes.create_string_buffer(1 << 16)
        nat.check(nat.lib().cgb_timing_report(self._h, buf, len(buf)), "cgb_timing_report")
        out = {}
        for line in buf.value.decode().splitlines():
            name, k, ms, b, mm = line.split()
            out[name] = (int(k), float(ms), float(b), float(mm))
        return out

    def modmul_peak(self) -> float:
        out = np.zeros(1, dtype=np.float64)
        nat.check(nat.lib().cgb_modmul_peak(self._h, nat.dblptr(out)), "cgb_modmul_peak")
        return float(out[0])

    def bench_ntt(self, count: int, fwd: bool, iters: int = 10) -> float:
        out = np.zeros(1, dtype=np.float64)
        nat.check(nat.lib().cgb_bench_ntt(self._h, int(count), int(fwd), int(iters), nat.dblptr(out)), "cgb_bench_ntt")
        return float(out[0])

    def sync(self):
        nat.check(nat.lib().cgb_sync(self._h), "cgb_sync")

    def set_stream(self, cuda_stream: int):
        nat.check(nat.lib().cgb_set_stream(self._h, ctypes.c_void_p(cuda_stream)), "cgb_set_stream")

    # storage -------------------------------------------------------------
    def alloc(self, n: int) -> np.ndarray:
        ids = np.zeros(n, dtype=np.uint32)
        if n:
            nat.check(nat.lib().cgb_ct_alloc(self._h, n, nat.u32ptr(ids)), "cgb_ct_alloc")
        return ids

    def free(self, ids):
        ids = _ids(ids)
        if ids.size and self._h:
            if self._ext:  # a freed ciphertext's extension goes with it (ids are reused)
                ext = [self._ext.pop(int(a)) for a in ids if int(a) in self._ext]
                if ext:
                    ids = np.concatenate([ids, np.concatenate(ext)]).astype(np.uint32)
            nat.check(nat.lib().cgb_ct_free(self._h, ids.size, nat.u32ptr(ids)), "cgb_ct_free")

    def ext_B(self, b_ids) -> np.ndarray:
        """Slot pairs of the base-B extensions of b_ids (2 per item), computing the
        missing ones; they live as long as their ciphertext's arena id."""
        b_ids = _ids(b_ids)
        missing = np.array(sorted({int(a) for a in b_ids} - self._ext.keys()), dtype=np.uint32)
        if missing.size:
            slots = self.alloc(2 * missing.size)
            nat.check(nat.lib().cgb_extend_b(self._h, missing.size, nat.u32ptr(missing), nat.u32ptr(slots)),
                      "cgb_extend_b")
            for k, a in enumerate(missing):
                self._ext[int(a)] = slots[2 * k:2 * k + 2].copy()
        return np.ascontiguousarray(np.concatenate([self._ext[int(a)] for a in b_ids]).astype(np.uint32))

    def free_slots(self) -> int:
        return int(nat.lib().cgb_ct_free_count(self._h))

    def has_ext(self, ids) -> bool:
        """Whether every id already has a resident base-B extension."""
        return bool(self._ext) and all(int(a) in self._ext for a in _ids(ids))

    def mult_cipher_ext(self, a, b, bx, out):
        a, b, bx, out = _ids(a), _ids(b), _ids(bx), _ids(out)
        nat.check(nat.lib().cgb_mult_cipher_ext(self._h, a.size, nat.u32ptr(a), nat.u32ptr(b), nat.u32ptr(bx),
                                                nat.u32ptr(out)), "cgb_mult_cipher_ext")

    def mult_cipher_ext2(self, a, ax, b, bx, out):
        """mult_cipher with both operands' base-B extensions resident (cgb_mult_cipher_ext2)."""
        a, ax, b, bx, out = _ids(a), _ids(ax), _ids(b), _ids(bx), _ids(out)
        nat.check(nat.lib().cgb_mult_cipher_ext2(self._h, a.size, nat.u32ptr(a), nat.u32ptr(ax), nat.u32ptr(b),
                                                 nat.u32ptr(bx), nat.u32ptr(out)), "cgb_mult_cipher_ext2")

    def alloc_pt(self, n: int) -> np.ndarray:
        ids = np.zeros(n, dtype=np.uint32)
        if n:
            nat.check(nat.lib().cgb_pt_alloc(self._h, n, nat.u32ptr(ids)), "cgb_pt_alloc")
        return ids

    def free_pt(self, ids):
        ids = _ids(ids)
        if ids.size and self._h:
            nat.check(nat.lib().cgb_pt_free(self._h, ids.size, nat.u32ptr(ids)), "cgb_pt_free")

    def copy(self, src, dst):
        src, dst = _ids(src), _ids(dst)
        nat.check(nat.lib().cgb_ct_copy(self._h, src.size, nat.u32ptr(src), nat.u32ptr(dst)), "cgb_ct_copy")

    def store(self, ids) -> np.ndarray:
        ids = _ids(ids)
        out = np.zeros((ids.size, 2, self.L, self.N), dtype=np.uint64)
        nat.check(nat.lib().cgb_ct_store(self._h, ids.size, nat.u32ptr(ids), nat.u64ptr(out)), "cgb_ct_store")
        return out

    def load(self, ids, words):
        ids = _ids(ids)
        w = np.ascontiguousarray(np.asarray(words, dtype=np.uint64).reshape(ids.size, 2, self.L, self.N))
        nat.check(nat.lib().cgb_ct_load(self._h, ids.size, nat.u32ptr(ids), nat.u64ptr(w)), "cgb_ct_load")

    # plaintexts ------------------------------------------------------------
    def _slots2d(self, slots, canonical: bool = False) -> np.ndarray:
        a = np.asarray(slots, dtype=np.int64)
        if a.ndim == 1:
            a = a.reshape(1, -1)
        if canonical:  # the caller's residues are in [0, t) by construction: no range pass
            return np.ascontiguousarray(a).view(np.uint64)
        if a.size and a.min() >= 0 and a.max() < self.t:  # already residues: zero-copy view
            return np.ascontiguousarray(a).view(np.uint64)
        return np.ascontiguousarray(np.mod(a, self.t).astype(np.uint64))

    def encode_pt(self, slots, kind: int, ids, canonical: bool = False):
        s, ids = self._slots2d(slots, canonical), _ids(ids)
        nat.check(nat.lib().cgb_pt_encode(self._h, ids.size, nat.u64ptr(s), kind, nat.u32ptr(ids)), "cgb_pt_encode")
        self.h2d_bytes += s.nbytes

    def mask_pcg64(self, chan_of_item, states, pt_neg=None, pt_pos=None, want_masks: bool = False):
        """Server masks drawn on the device (cgb_mask_pcg64): item i takes the next
        n_slots words of channel chan_of_item[i]'s numpy PCG64 stream; ``states``
        (uint64[nchan][6]) is advanced in place.  Returns the masks when asked."""
        ch = np.ascontiguousarray(np.asarray(chan_of_item, dtype=np.int32))
        st = states
        assert st.dtype == np.uint64 and st.flags.c_contiguous and st.shape[1] == 6
        out = np.zeros((ch.size, self.n_slots), np.uint64) if want_masks else None
        nat.check(nat.lib().cgb_mask_pcg64(self._h, ch.size, st.shape[0],
                                           ch.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), nat.u64ptr(st),
                                           None if pt_neg is None else nat.u32ptr(_ids(pt_neg)),
                                           None if pt_pos is None else nat.u32ptr(_ids(pt_pos)),
                                           None if out is None else nat.u64ptr(out)), "cgb_mask_pcg64")
        return None if out is None else out.view(np.int64)

    # client role -----------------------------------------------------------
    def encrypt(self, slots, enc_key, first_index: int, ids):
        s, ids = self._slots2d(slots), _ids(ids)
        k = np.ascontiguousarray(np.asarray(enc_key, dtype=np.uint32).reshape(8))
        nat.check(nat.lib().cgb_encrypt(self._h, ids.size, nat.u64ptr(s), nat.u32ptr(k), int(first_index),
                                        nat.u32ptr(ids)), "cgb_encrypt")
        self.h2d_bytes += s.nbytes

    def encrypt_batch(self, slots, enc_keys, indices, ids, canonical: bool = False):
        """Item i encrypted with key enc_keys[i] (8 words) at encryption index indices[i]."""
        s, ids = self._slots2d(slots, canonical), _ids(ids)
        k = np.ascontiguousarray(np.asarray(enc_keys, dtype=np.uint32).reshape(ids.size, 8))
        ix = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64).reshape(ids.size))
        nat.check(nat.lib().cgb_encrypt_batch(self._h, ids.size, nat.u64ptr(s), nat.u32ptr(k), nat.u64ptr(ix),
                                              nat.u32ptr(ids)), "cgb_encrypt_batch")
        self.h2d_bytes += s.nbytes

    def reencrypt_batch(self, src, enc_keys, indices, out):
        """Decrypt each src item and encrypt its slots again (key enc_keys[i], index
        indices[i]) without leaving the device (cgb_reencrypt_batch)."""
        src, out = _ids(src), _ids(out)
        k = np.ascontiguousarray(np.asarray(enc_keys, dtype=np.uint32).reshape(src.size, 8))
        ix = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64).reshape(src.size))
        nat.check(nat.lib().cgb_reencrypt_batch(self._h, src.size, nat.u32ptr(src), nat.u32ptr(k), nat.u64ptr(ix),
                                                nat.u32ptr(out)), "cgb_reencrypt_batch")

    def decrypt(self, ids) -> np.ndarray:
        ids = _ids(ids)
        out = np.zeros((ids.size, self.n_slots), dtype=np.uint64)
        nat.check(nat.lib().cgb_decrypt(self._h, ids.size, nat.u32ptr(ids), nat.u64ptr(out)), "cgb_decrypt")
        self.d2h_bytes += out.nbytes
        return out.view(np.int64)  # residues < t < 2^63: the same values, no copy

    def decrypt_start(self, ids):
        """Enqueue a decryption (and its device->host copy straight into a
        page-locked array); returns a ticket for decrypt_finish.  Only that ticket
        is waited for."""
        from .nonlinear import host_buffer  # page-locked up to 128 MB (torch's caching host allocator)

        ids = _ids(ids)
        # always page-locked when it fits: a copy into pageable memory would make this
        # call wait for everything queued before it
        out = host_buffer((ids.size, self.n_slots), min_words=0)
        t = ctypes.c_void_p()
        nat.check(nat.lib().cgb_decrypt_start_into(self._h, ids.size, nat.u32ptr(ids),
                                                   out.ctypes.data_as(nat._u64p), ctypes.byref(t)),
                  "cgb_decrypt_start_into")
        return t, out

    def decrypt_finish(self, ticket) -> np.ndarray:
        t, out = ticket
        nat.check(nat.lib().cgb_decrypt_finish(self._h, t, None), "cgb_decrypt_finish")
        self.d2h_bytes += out.nbytes
        return out  # residues < t < 2^63 as int64, page-locked (later uploads are DMA)

    def noise_budget(self, ids) -> np.ndarray:
        ids = _ids(ids)
        out = np.zeros(ids.size, dtype=np.float64)
        nat.check(nat.lib().cgb_noise_budget(self._h, ids.size, nat.u32ptr(ids), nat.dblptr(out)), "cgb_noise_budget")
        return out

    # server role -----------------------------------------------------------
    def _bin(self, fn, what, a, b, out):
        a, b, out = _ids(a), _ids(b), _ids(out)
        nat.check(fn(self._h, a.size, nat.u32ptr(a), nat.u32ptr(b), nat.u32ptr(out)), what)

    def add(self, a, b, out):
        self._bin(nat.lib().cgb_add, "cgb_add", a, b, out)

    def add_plain(self, a, pt, out):
        self._bin(nat.lib().cgb_add_plain, "cgb_add_plain", a, pt, out)

    def mult_plain(self, a, pt, out):
        self._bin(nat.lib().cgb_mult_plain, "cgb_mult_plain", a, pt, out)

    def mult_cipher(self, a, b, out):
        self._bin(nat.lib().cgb_mult_cipher, "cgb_mult_cipher", a, b, out)

    def galois(self, a, gs, out):
        a, out = _ids(a), _ids(out)
        g = np.ascontiguousarray(np.broadcast_to(np.asarray(gs, dtype=np.uint64), a.shape))
        nat.check(nat.lib().cgb_galois(self._h, a.size, nat.u32ptr(a), nat.u64ptr(g), nat.u32ptr(out)), "cgb_galois")

    def rotate(self, a, steps, out, add_input: bool = False):
        a, out = _ids(a), _ids(out)
        st = np.ascontiguousarray(np.broadcast_to(np.asarray(steps, dtype=np.int64), a.shape))
        fn = nat.lib().cgb_rotate_add if add_input else nat.lib().cgb_rotate
        nat.check(fn(self._h, a.size, nat.u32ptr(a), nat.i64ptr(st), nat.u32ptr(out)), "cgb_rotate")

    def rotate_add_chain(self, a, steps, out):
        """x <- x + rotate(x, s) for s in steps, in one call (intermediates in scratch)."""
        a, out = _ids(a), _ids(out)
        st = np.ascontiguousarray(np.asarray(steps, dtype=np.int64).reshape(-1))
        nat.check(nat.lib().cgb_rotate_add_chain(self._h, a.size, nat.u32ptr(a), st.size, nat.i64ptr(st),
                                                 nat.u32ptr(out)), "cgb_rotate_add_chain")

    def sum(self, a, out: int):
        a = _ids(a)
        nat.check(nat.lib().cgb_sum(self._h, a.size, nat.u32ptr(a), int(out)), "cgb_sum")

    def prepare_galois(self, gs):
        g = np.ascontiguousarray(np.asarray(gs, dtype=np.uint64).reshape(-1))
        nat.check(nat.lib().cgb_prepare_galois(self._h, g.size, nat.u64ptr(g)), "cgb_prepare_galois")

    def galois_elt(self, k: int) -> int:
        return pow(5, int(k) % (self.n_slots if self.one_row else self.n_slots // 2), 2 * self.N)
