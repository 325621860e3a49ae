"""Loader for the sm_100a backend library ``libcgb200.so`` (include/cgb200.h).

There is no fallback: if the library or a CUDA device is missing every
entry point raises ``BackendUnavailable``.  ``build()`` compiles the
library in-tree with nvcc for sm_100a.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SO_PATH = PKG / "libcgb200.so"
SOURCES = [PKG / "csrc" / "cgb200.cu", PKG / "csrc" / "cgb_device.cuh", PKG / "csrc" / "cgb_masks.cuh",
           ROOT / "include" / "cgb200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]

CGB_OK, CGB_ERR_PARAM, CGB_ERR_CUDA, CGB_ERR_NOMEM, CGB_ERR_STATE = range(5)
CGB_PT_MUL, CGB_PT_ADD = 0, 1


class BackendUnavailable(RuntimeError):
    """The CUDA backend library could not be loaded or has no device."""


class BackendError(RuntimeError):
    """A runtime failure reported by the backend library."""


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile libcgb200.so in-tree (no-op when newer than its sources)."""
    newest = max(p.stat().st_mtime for p in SOURCES)
    if not force and SO_PATH.exists() and SO_PATH.stat().st_mtime >= newest:
        return SO_PATH
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-o", str(SO_PATH), str(SOURCES[0])]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return SO_PATH


_lib = None

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_dblp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p

SIGNATURES = {
    "cgb_ring_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       _u32p, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(_vp)]),
    "cgb_ring_create_ex": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, _u32p, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(_vp)]),
    "cgb_ring_destroy": (None, [_vp]),
    "cgb_ring_moduli": (ctypes.c_int, [_vp, _u64p, ctypes.c_int]),
    "cgb_ct_words": (ctypes.c_size_t, [_vp]),
    "cgb_last_error": (ctypes.c_char_p, []),
    "cgb_set_stream": (ctypes.c_int, [_vp, _vp]),
    "cgb_sync": (ctypes.c_int, [_vp]),
    "cgb_launch_count": (ctypes.c_uint64, [_vp]),
    "cgb_timing_enable": (ctypes.c_int, [_vp, ctypes.c_int]),
    "cgb_timing_report": (ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_size_t]),
    "cgb_modmul_peak": (ctypes.c_int, [_vp, _dblp]),
    "cgb_bench_ntt": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dblp]),
    "cgb_ct_alloc": (ctypes.c_int, [_vp, ctypes.c_int, _u32p]),
    "cgb_ct_free": (ctypes.c_int, [_vp, ctypes.c_int, _u32p]),
    "cgb_ct_copy": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u32p]),
    "cgb_ct_store": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u64p]),
    "cgb_ct_load": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u64p]),
    "cgb_ct_device_ptr": (_u64p, [_vp, ctypes.c_uint32]),
    "cgb_pt_alloc": (ctypes.c_int, [_vp, ctypes.c_int, _u32p]),
    "cgb_pt_free": (ctypes.c_int, [_vp, ctypes.c_int, _u32p]),
    "cgb_pt_encode": (ctypes.c_int, [_vp, ctypes.c_int, _u64p, ctypes.c_int, _u32p]),
    "cgb_ct_free_count": (ctypes.c_int64, [_vp]),
    "cgb_reencrypt_batch": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u32p, _u64p, _u32p]),
    "cgb_mult_cipher_ext2": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u32p, _u32p, _u32p, _u32p]),
    "cgb_mask_pcg64": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int32), _u64p, _u32p,
                                      _u32p, _u64p]),
    "cgb_encrypt": (ctypes.c_int, [_vp, ctypes.c_int, _u64p, _u32p, ctypes.c_uint64, _u32p]),
    "cgb_encrypt_batch": (ctypes.c_int, [_vp, ctypes.c_int, _u64p, _u32p, _u64p, _u32p]),
    "cgb_decrypt": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u64p]),
    "cgb_decrypt_start": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, ctypes.POINTER(_vp)]),
    "cgb_decrypt_finish": (ctypes.c_int, [_vp, _vp, _u64p]),
    "cgb_decrypt_start_into": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u64p, ctypes.POINTER(_vp)]),
    "cgb_noise_budget": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _dblp]),
    "cgb_add": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u32p, _u32p]),
    "cgb_add_plain": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u32p, _u32p]),
    "cgb_mult_plain": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u32p, _u32p]),
    "cgb_mult_cipher": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u32p, _u32p]),
    "cgb_extend_b": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u32p]),
    "cgb_mult_cipher_ext": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u32p, _u32p, _u32p]),
    "cgb_galois": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _u64p, _u32p]),
    "cgb_rotate": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _i64p, _u32p]),
    "cgb_rotate_add": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, _i64p, _u32p]),
    "cgb_rotate_add_chain": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, ctypes.c_int, _i64p, _u32p]),
    "cgb_sum": (ctypes.c_int, [_vp, ctypes.c_int, _u32p, ctypes.c_uint32]),
    "cgb_prepare_galois": (ctypes.c_int, [_vp, ctypes.c_int, _u64p]),
}


def load_library(path: Path | None = None):
    """dlopen the library and bind every symbol of include/cgb200.h.

    Works without a GPU (symbol checks); compute calls need a device."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # CGB_LIB: an alternative in-tree build of the same library (build-variant experiments)
    p = Path(path) if path else Path(os.environ.get("CGB_LIB", SO_PATH))
    if not p.exists():
        raise BackendUnavailable(
            f"{p} is missing: run __graft_entry__.build() (nvcc, sm_100a) first"
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def lib():
    return load_library()


def check(rc: int, what: str = ""):
    if rc == CGB_OK:
        return
    msg = (lib().cgb_last_error() or b"").decode(errors="replace")
    if rc == CGB_ERR_PARAM:
        from .backend import ParameterError

        raise ParameterError(f"{what}: {msg}")
    raise BackendError(f"{what}: {msg} (code {rc})")


def u32ptr(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(_u32p)


def u64ptr(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(_u64p)


def i64ptr(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def dblptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dblp)
