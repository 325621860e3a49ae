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


@pytest.mark.parametrize("spec,n_items,rounds", [((14, 536903681, 3, 8192, True, 49), 24, 40),
                                                 ((7, 67109633, 4, 64, True, 60), 512, 1200)],
                         ids=["bench_ring", "toy_ring_wraps_staging"])
def test_stream_switches_between_calls_keep_results(spec, n_items, rounds):
    """The pointer tables of a call are uploaded on a side stream into a device mirror of
    the pinned staging area and the compute stream waits for the upload's event.  Many
    small calls, the ring's stream switched between them (cgb_set_stream), wrap the
    staging halves several times; every output must equal the single-stream run."""
    import torch

    from paper_2602_08798_b200._native import build
    from paper_2602_08798_b200.ring import Ring

    build()
    key = np.arange(8, dtype=np.uint32) * 3 + 1
    enc = np.arange(8, dtype=np.uint32) + 77
    log_n, t, L, n, one_row, qb = spec

    def run(streams):
        # (the toy ring's staging area is 8 MB: 1200 uploads of 16 KB wrap its halves twice)
        g = Ring(log_n, t, L, n, one_row, key, arena_cts=4 * n_items + 8, arena_pts=8, q_bits=qb)
        rng = np.random.default_rng(9)
        src = g.alloc(n_items)
        g.encrypt(rng.integers(0, t, (n_items, n)), enc, 0, src)
        a, b = src, g.alloc(n_items)
        for r in range(rounds):
            s = streams[r % len(streams)]
            if s is not None:
                # hand over: the next stream waits for everything queued so far
                prev = streams[(r - 1) % len(streams)]
                if prev is not None and prev is not s:
                    s.wait_stream(prev)
                g.set_stream(s.cuda_stream)
            steps = (np.arange(1, n_items + 1, dtype=np.int64) * (r + 1)) % n
            steps[steps == 0] = 1
            g.rotate(a, steps, b, add_input=bool(r & 1))
            a, b = b, (g.alloc(n_items) if a is src else a)
        torch.cuda.synchronize()
        return g.store(a)

    one = run([None])
    two = run([torch.cuda.Stream(), torch.cuda.Stream()])
    assert np.array_equal(one, two)
