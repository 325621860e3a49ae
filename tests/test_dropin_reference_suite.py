"""The drop-in, proven with the reference's own tests.

``dropin.install()`` swaps ``cryptogen.backend.Context`` (the reference's
only substrate, /root/reference/pkg/src/cryptogen/backend.py:245-368) for
the B200 context.  The GPU test runs the UNMODIFIED reference test files
(installed next to the package in baseline/_ref by
scripts/install_reference.sh; skipped when absent) with every context on
the GPU ring, and requires them all to pass.
"""
import json
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
SUITE = REF / "cryptogen_tests"
# the substrate, packing, kernel, cache and share-conversion suites (the hot path's
# reference tests; test_acceptance / test_model / test_cli drive the toy model and CLI)
FILES = ["test_backend.py", "test_encodings.py", "test_linear_kernels.py", "test_arcc.py", "test_kv_cache.py",
         "test_nonlinear.py"]

needs_ref = pytest.mark.skipif(not (REF / "cryptogen").is_dir() or not SUITE.is_dir(),
                               reason="reference not installed (scripts/install_reference.sh)")


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT), str(ROOT / "tests"), env.get("PYTHONPATH", "")])
    return env


@needs_ref
def test_install_rebinds_every_reference_binding():
    """install() rebinds the package-root re-exports, cli.py's by-name import and
    the exception classes this package raises (no context is created: CPU)."""
    code = r"""
import sys, json
import cryptogen, cryptogen.backend as rb, cryptogen.cli as cli
old = rb.new_context
from paper_2602_08798_b200 import dropin, backend, kv_cache, arcc, model
C = dropin.install()
assert dropin.install() is C
out = {
  "backend": rb.Context is C, "root_ctx": cryptogen.Context is C if hasattr(cryptogen, "Context") else True,
  "root_new": cryptogen.new_context is rb.new_context, "cli_new": cli.new_context is rb.new_context,
  "changed": rb.new_context is not old,
  "errors": all(getattr(m, "ParameterError") is rb.ParameterError for m in (backend, kv_cache, arcc, model)),
  "budget_err": backend.NoiseBudgetExhausted is rb.NoiseBudgetExhausted,
  "subclass": issubclass(C, backend.GpuContext),
}
print(json.dumps(out))
"""
    res = subprocess.run([sys.executable, "-c", code], env=_env(), capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-3000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert all(out.values()), out


@pytest.mark.gpu
@needs_ref
def test_reference_suite_passes_on_gpu_context():
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "ref_dropin_plugin", "-p", "no:cacheprovider",
           "--rootdir", str(SUITE), "-o", "addopts=", *[str(SUITE / f) for f in FILES]]
    res = subprocess.run(cmd, env=_env(), capture_output=True, text=True, timeout=3000, cwd=str(SUITE))
    tail = res.stdout[-4000:]
    print(tail)
    m = re.search(r"(\d+) passed", tail)
    assert res.returncode == 0 and m, tail + res.stderr[-2000:]
    assert "GPU contexts created" in tail and "dropin: cryptogen.backend.Context is paper_2602_08798_b200" in tail
    out = os.environ.get("CGB_REF_SUITE_OUT")
    if out:
        Path(out).write_text(json.dumps({"files": FILES, "passed": int(m.group(1)), "summary": tail[-600:]}))
