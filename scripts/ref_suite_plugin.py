"""pytest plugin: run the reference's own test suite with cryptogen.backend.Context
replaced by the B200 GPU context (the drop-in claim)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))


def pytest_configure(config):
    from paper_2602_08798_b200 import _native, dropin

    _native.build()
    dropin.install()
