"""Install the B200 backend under an existing ``cryptogen`` installation.

The reference resolves its substrate through ``cryptogen.backend.Context``
at call time (``new_context`` backend.py:367-368, ``Context.fork`` :278-280),
so swapping that one name moves every kernel of the reference package --
encodings, linear kernels, arcc, kv_cache, nonlinear, model -- onto the GPU
ring, unmodified.  The exception classes are unified so the reference's
``except`` clauses and tests see the errors they expect.

    import cryptogen
    from paper_2602_08798_b200 import dropin
    dropin.install()          # cryptogen.backend.Context -> GpuContext

The head-batched fused paths (``attention_step_heads`` etc.) are called
through this package's own modules, which mirror the reference's names.
"""
from __future__ import annotations

import sys

from . import backend as _b

_MODULES = ("backend", "encodings", "linear_kernels", "arcc", "kv_cache", "nonlinear", "fixedpoint", "_native")


def install(cryptogen_backend=None):
    """Point ``cryptogen.backend.Context`` / ``new_context`` at the GPU context."""
    if cryptogen_backend is None:
        import cryptogen.backend as cryptogen_backend  # noqa: PLW0621
    rb = cryptogen_backend
    # one set of exception classes across both packages
    for name in ("ParameterError", "NoiseBudgetExhausted", "DecryptionFailure"):
        ref_cls = getattr(rb, name)
        for mod in _MODULES:
            m = sys.modules.get(f"{__package__}.{mod}")
            if m is not None and hasattr(m, name):
                setattr(m, name, ref_cls)

    class Context(_b.GpuContext):
        """cryptogen Context realised on the B200 RNS-BFV ring."""

        def fork(self):
            return Context(self.params, self._seed_seq.spawn(1)[0], self._n_limbs)

    rb.Context = Context
    rb.new_context = lambda params, seed=0: Context(params, seed)
    return Context
