"""Concurrent use of one ring from several threads.

The reference runs attention heads on a thread pool, one forked context per
thread (model.py:395-400, :420-442).  Forked GPU contexts
share their ring (keys, arenas, staging buffers), so the library serialises
the ring's entry points; results must equal the serial run.
"""
import concurrent.futures as cf

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p", [(64, 67109633), (8192, 536903681)])
def test_threads_on_forked_contexts_equal_serial(n, p):
    from paper_2602_08798_b200._native import build
    from paper_2602_08798_b200.backend import BackendParams, GpuContext

    build()

    def work(ctx, seed):
        rng = np.random.default_rng(seed)
        a = ctx.encrypt(rng.integers(0, p, n))
        b = ctx.encrypt(rng.integers(0, p, n))
        x = ctx.mult_cipher(ctx.rotate(a, 3), b)
        for k in (1, 2, 4, 8):
            x = ctx.add(x, ctx.rotate(x, k))
        x = ctx.mult_plain(x, rng.integers(0, p, n))
        return ctx.decrypt(x), x.words()

    outs = {}
    for threads in (1, 6):
        root = GpuContext(BackendParams(n_slots=n, plain_modulus=p), 5)
        ctxs = [root.fork() for _ in range(12)]
        if threads == 1:
            outs[threads] = [work(c, i) for i, c in enumerate(ctxs)]
        else:
            with cf.ThreadPoolExecutor(threads) as ex:
                outs[threads] = list(ex.map(lambda ic: work(ic[1], ic[0]), enumerate(ctxs)))
    for (d1, w1), (d6, w6) in zip(outs[1], outs[6]):
        assert np.array_equal(d1, d6)
        assert np.array_equal(w1, w6)
