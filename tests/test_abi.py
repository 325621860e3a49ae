"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
entry point include/cgb200.h declares (no compute calls)."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def declared():
    text = (ROOT / "include" / "cgb200.h").read_text()
    return sorted(set(re.findall(r"\b(cgb_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    for need in ("cgb_ring_create", "cgb_encrypt", "cgb_decrypt", "cgb_add", "cgb_add_plain", "cgb_mult_plain",
                 "cgb_mult_cipher", "cgb_rotate", "cgb_galois", "cgb_rotate_add", "cgb_rotate_add_chain"):
        assert need in names


def test_library_exports_every_declared_symbol():
    from paper_2602_08798_b200 import _native

    _native.build()
    lib = _native.load_library()
    for name in declared():
        assert hasattr(lib, name), name
    # the Python binding table covers the header exactly
    assert set(_native.SIGNATURES) == set(declared())


def test_library_is_sm100a():
    import subprocess

    from paper_2602_08798_b200 import _native

    so = _native.build()
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_means_loud_failure(monkeypatch):
    """Without a device the backend raises instead of silently falling back."""
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2602_08798_b200 import BackendParams, new_context

    with pytest.raises(Exception):
        new_context(BackendParams(n_slots=16, plain_modulus=97), 0)
