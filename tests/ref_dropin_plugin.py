"""pytest plugin: run the reference's own test suite on the GPU context.

Loaded with ``-p ref_dropin_plugin`` BEFORE the reference's conftest
(/root/reference/pkg/tests/conftest.py:4 imports ``new_context`` by name),
it imports the unmodified reference package from ``baseline/_ref`` and
calls ``paper_2602_08798_b200.dropin.install()``, so every context the
reference's tests create is the B200 RNS-BFV context.  Used by
tests/test_dropin_reference_suite.py; never by the product.
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
for p in (str(REF), str(ROOT)):
    if p not in sys.path:
        sys.path.insert(0, p)

import cryptogen  # noqa: E402,F401
import cryptogen.backend  # noqa: E402

from paper_2602_08798_b200 import dropin  # noqa: E402

GPU_CONTEXT = dropin.install()
_made = []


def pytest_configure(config):
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the drop-in suite runs on the GPU context: no CUDA device")
    orig_init = GPU_CONTEXT.__init__

    def counting_init(self, *a, **kw):
        orig_init(self, *a, **kw)
        _made.append(1)

    GPU_CONTEXT.__init__ = counting_init


def pytest_terminal_summary(terminalreporter):
    import cryptogen.backend as rb

    terminalreporter.write_line(
        f"dropin: cryptogen.backend.Context is {rb.Context.__module__}.{rb.Context.__qualname__}; "
        f"{len(_made)} GPU contexts created")
