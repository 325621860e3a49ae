"""Install the B200 backend under an existing ``cryptogen`` installation.

The reference resolves its substrate through ``cryptogen.backend.Context``
at call time (``new_context`` backend.py:367-368, ``Context.fork`` :278-280),
so swapping that name moves every kernel of the reference package --
encodings, linear kernels, arcc, kv_cache, nonlinear, model -- onto the GPU
ring, unmodified.  Names bound by value elsewhere are rebound too: the
package root's re-exports (cryptogen/__init__.py:11-22), ``cli.py``'s
``from .backend import new_context`` (cli.py:20) and any already-imported
module holding the old objects.  The exception classes are unified (every
module of this package raises the reference's classes) and counters are the
reference's ``OpCounter`` (backend.py:173-213), so the reference's
``except`` clauses, ``pytest.raises`` and counter comparisons see what they
expect.

    import cryptogen
    from paper_2602_08798_b200 import dropin
    dropin.install()          # cryptogen.backend.Context -> GPU context

Modules imported AFTER install() that bind ``new_context`` by name get the
GPU one (they read it from cryptogen.backend).  tests/ref_dropin_plugin.py
installs this before the reference's own test suite is imported and runs it
on the GPU (tests/test_dropin_reference_suite.py).
"""
from __future__ import annotations

import sys

from . import backend as _b

_ERRORS = ("ParameterError", "NoiseBudgetExhausted", "DecryptionFailure")
_installed = None


def install(cryptogen_backend=None):
    """Point every ``cryptogen`` binding of ``Context`` / ``new_context`` at the
    GPU context; returns the installed Context class (idempotent)."""
    global _installed
    if cryptogen_backend is None:
        import cryptogen.backend as cryptogen_backend  # noqa: PLW0621
    rb = cryptogen_backend
    if _installed is not None and rb.Context is _installed:
        return _installed
    # one set of exception classes across both packages: every loaded module of this
    # package raises the reference's classes from now on
    for modname, m in list(sys.modules.items()):
        if m is None or not (modname == __package__ or modname.startswith(__package__ + ".")):
            continue
        for name in _ERRORS:
            if hasattr(m, name):
                setattr(m, name, getattr(rb, name))

    ref_counter = rb.OpCounter

    class Context(_b.GpuContext):
        """cryptogen Context realised on the B200 RNS-BFV ring."""

        def __init__(self, params, seed=0, n_limbs=None):
            super().__init__(params, seed, n_limbs)
            self.counter = ref_counter()

        def fork(self):
            return Context(self.params, self._seed_seq.spawn(1)[0], self._n_limbs)

    def new_context(params, seed=0):
        return Context(params, seed)

    old_ctx, old_new = rb.Context, rb.new_context
    rb.Context, rb.new_context = Context, new_context
    # by-value bindings: cryptogen/__init__.py re-exports, cli.py, any loaded module
    for modname, m in list(sys.modules.items()):
        if m is None or not (modname == "cryptogen" or modname.startswith("cryptogen.")) or m is rb:
            continue
        if getattr(m, "Context", None) is old_ctx:
            setattr(m, "Context", Context)
        if getattr(m, "new_context", None) is old_new:
            setattr(m, "new_context", new_context)
    _installed = Context
    return Context
