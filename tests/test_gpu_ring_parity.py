"""Word-exact parity of the kernels the bench times, on the benchmarked ring.

The decode bench (bench.py) runs N = 16384, L = 3 primes < 2^49, n = 8192
slots, p = 536903681 -- the instantiations keyswitch_fp_t<7,7,3>,
k_ks_row<7,7,3,*>, keyswitch_hoisted_t<7,7,3> and the FP64 base
conversions of mult_cipher.  Here every output word of batched waves of
>= 256 ciphertexts (per-item Galois elements) is compared with the CPU
RNS-BFV oracle (oracle/rnsbfv.c), and one whole decode attention step of
the reference's op sequence (oracle/reference_path.py over
oracle/rns_context.py, i.e. /root/reference/pkg/src/cryptogen/
arcc.py:320-379 op by op) is compared with the fused head-batched wave
schedule (arcc.attention_step_heads) ciphertext word for ciphertext word.
"""
import concurrent.futures as cf
import os
import sys
import threading
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))

KEY = np.arange(8, dtype=np.uint32) * 7 + 1
ENC = np.arange(8, dtype=np.uint32) + 1000
BENCH_RING = (14, 536903681, 3, 8192, True, 49)
COUNT = 256
WORKERS = max(1, min(16, os.cpu_count() or 1))


class OraclePool:
    """One OracleRing per worker thread (the C oracle caches keys per ring;
    ctypes drops the GIL, so the scalar oracle runs in parallel)."""

    def __init__(self, mod, spec, key):
        self.mod, self.spec, self.key = mod, spec, key
        self.local = threading.local()
        self.ex = cf.ThreadPoolExecutor(WORKERS)

    def ring(self):
        r = getattr(self.local, "r", None)
        if r is None:
            log_n, t, L, n, one_row, qb = self.spec
            r = self.local.r = self.mod.OracleRing(log_n, t, L, n, one_row, self.key, q_bits=qb)
        return r

    def map(self, fn, *its):
        return list(self.ex.map(lambda args: fn(self.ring(), *args), zip(*its)))


@pytest.fixture(scope="module")
def bench(oracle_mod):
    from paper_2602_08798_b200._native import build
    from paper_2602_08798_b200.ring import Ring

    build()
    log_n, t, L, n, one_row, qb = BENCH_RING
    g = Ring(log_n, t, L, n, one_row, KEY, arena_cts=6 * COUNT + 64, arena_pts=64, q_bits=qb)
    pool = OraclePool(oracle_mod, BENCH_RING, KEY)
    rng = np.random.default_rng(2024)
    vals = rng.integers(0, t, (COUNT, n))
    ids = g.alloc(COUNT)
    g.encrypt(vals, ENC, 0, ids)
    words = g.store(ids)
    return g, pool, vals, ids, words


def test_batched_encrypt_bitexact(bench):
    g, pool, vals, ids, words = bench
    sel = np.arange(0, COUNT, 17)  # every 17th item (encryption is covered item by item elsewhere)
    want = pool.map(lambda o, v, i: o.encrypt(v, ENC, int(i)), vals[sel], sel)
    for k, i in enumerate(sel):
        assert np.array_equal(words[i], want[k]), i


@pytest.mark.parametrize("add", [False, True], ids=["rotate", "rotate_add"])
def test_batched_rotate_bitexact(bench, add):
    """256 distinct sources, 256 distinct steps (one Galois key each): the
    five-launch fused key switch (cgb_rotate / cgb_rotate_add)."""
    g, pool, vals, ids, words = bench
    n = g.n_slots
    steps = np.random.default_rng(7).choice(n, COUNT, replace=False).astype(np.int64)
    out = g.alloc(COUNT)
    g.rotate(ids, steps, out, add_input=add)
    got = g.store(out)
    g.free(out)

    def ref(o, w, k):
        r = o.rotate(w, int(k))
        return o.add(r, w) if add else r

    want = pool.map(ref, words, steps)
    bad = [i for i in range(COUNT) if not np.array_equal(got[i], want[i])]
    assert not bad, f"{len(bad)} items differ, first {bad[:8]}"


def test_rotate_add_chain_bitexact(bench):
    """cgb_rotate_add_chain (a fold's doubling steps in one call, intermediates in
    scratch) against the oracle's step-by-step rotate + add, every word; also equal to
    the same steps issued one cgb_rotate_add at a time, including in-place output."""
    g, pool, vals, ids, words = bench
    cnt = 12
    steps = [1, 2, 4, -64, 8191]
    out = g.alloc(cnt)
    g.rotate_add_chain(ids[:cnt], steps, out)
    got = g.store(out)

    def ref(o, w):
        for k in steps:
            w = o.add(o.rotate(w, int(k)), w)
        return w

    want = pool.map(ref, words[:cnt])
    for i in range(cnt):
        assert np.array_equal(got[i], want[i]), i
    # step by step through the arena, and a one-step chain
    cur = ids[:cnt]
    tmp = []
    for k in steps:
        nxt = g.alloc(cnt)
        g.rotate(cur, np.full(cnt, k, np.int64), nxt, add_input=True)
        tmp.append(nxt)
        cur = nxt
    assert np.array_equal(g.store(cur), got)
    one = g.alloc(cnt)
    g.rotate_add_chain(ids[:cnt], steps[:1], one)
    assert np.array_equal(g.store(one), g.store(tmp[0]))
    for t in tmp + [one, out]:
        g.free(t)


def test_wave_chain_equals_step_loop():
    """GpuContext.w_rotate_add_chain charges counters, ids and budgets exactly as the
    loop of w_rotate(add_input=True) does, and yields the same words."""
    import paper_2602_08798_b200 as cg
    from paper_2602_08798_b200 import backend

    def run(chain):
        backend._ROT_CHAIN = chain
        ctxs = [cg.new_context(cg.BackendParams(n_slots=8192, plain_modulus=536903681), seed=s) for s in (1, 2)]
        rng = np.random.default_rng(5)
        C = type(ctxs[0])
        owners = [ctxs[0], ctxs[1], ctxs[0], ctxs[1], ctxs[1]]
        w = C.w_encrypt(owners, rng.integers(0, 536903681, (5, 8192)))
        w = C.w_rotate_add_chain(w, [1, 2, 4, 8])
        words = ctxs[0]._ring.store(w.aids)
        # ciphertext ids carry a per-context base (a multiple of 10^9): compare the sequence numbers
        return (words, w.budgets.copy(), w.cids % 10**9,
                [(c.counter.rotate, c.counter.add, c._next_id % 10**9) for c in ctxs])

    try:
        a, b = run(True), run(False)
    finally:
        backend._ROT_CHAIN = True
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) and a[3] == b[3]


def test_batched_rotate_decrypts(bench):
    g, pool, vals, ids, words = bench
    steps = np.array([1, 2, 4095, 4096, 8191, 100], np.int64)
    out = g.alloc(steps.size)
    g.rotate(ids[: steps.size], steps, out)
    dec = g.decrypt(out)
    for i, k in enumerate(steps):
        assert np.array_equal(dec[i], np.roll(vals[i], -int(k)))
    g.free(out)


@pytest.mark.parametrize("add", [False, True], ids=["hoisted", "hoisted_add"])
def test_batched_rotate_hoisted_bitexact(bench, add):
    """8 sources x 32 steps each (the CPVM diagonal pattern): one ModUp per
    source, per-item Galois gathers (keyswitch_hoisted_t, k_ks_inner_hoist)."""
    g, pool, vals, ids, words = bench
    n = g.n_slots
    src_idx = np.repeat(np.arange(8), COUNT // 8)
    steps = np.random.default_rng(8).choice(n, COUNT, replace=False).astype(np.int64)
    out = g.alloc(COUNT)
    g.rotate(ids[src_idx], steps, out, add_input=add)
    got = g.store(out)
    g.free(out)

    def ref(o, s, k):
        r = o.rotate(words[s], int(k))
        return o.add(r, words[s]) if add else r

    want = pool.map(ref, src_idx, steps)
    bad = [i for i in range(COUNT) if not np.array_equal(got[i], want[i])]
    assert not bad, f"{len(bad)} items differ, first {bad[:8]}"


def test_batched_mult_cipher_bitexact(bench):
    """256 products (HPS tensor, FP64 base conversions, relinearisation), and
    the same with b's base-B extension resident (cgb_mult_cipher_ext)."""
    g, pool, vals, ids, words = bench
    b_idx = np.roll(np.arange(COUNT), 1)
    out = g.alloc(2 * COUNT)
    g.mult_cipher(ids, ids[b_idx], out[:COUNT])
    g.mult_cipher_ext(ids, ids[b_idx], g.ext_B(ids[b_idx]), out[COUNT:])
    got = g.store(out)
    want = pool.map(lambda o, i, j: o.mult_cipher(words[i], words[j]), np.arange(COUNT), b_idx)
    bad = [i for i in range(COUNT) if not np.array_equal(got[i], want[i])]
    assert not bad, f"mult_cipher: {len(bad)} items differ, first {bad[:8]}"
    bad = [i for i in range(COUNT) if not np.array_equal(got[COUNT + i], want[i])]
    assert not bad, f"mult_cipher_ext: {len(bad)} items differ, first {bad[:8]}"
    dec = g.decrypt(out[:4])
    for i in range(4):
        assert np.array_equal(dec[i], vals[i] * vals[b_idx[i]] % g.t)
    g.free(out)


def test_attention_step_words_equal_reference_sequence(oracle_mod):
    """One decode attention step, 2 heads, n = 8192, d2 = 4, m = 5, t = 3 on
    the production ring: the B200 wave schedule against the reference's op
    sequence executed op by op on the CPU RNS-BFV oracle.  Every output
    ciphertext word, every counter and every transcript entry must agree."""
    import harness
    from hostapi import repo_api
    from oracle import reference_path as ref
    from oracle.rns_context import OracleContext
    from paper_2602_08798_b200 import backend as B
    from paper_2602_08798_b200._native import build

    build()
    api = repo_api()
    n, p, d2, m, t, H, seed = 8192, harness.P8192, 4, 5, 3, 2, 21
    root, fp, ctxs, caches, qs, chans = harness.attention_heads(api, B.GpuContext, n, p, d2, m, t, H, seed=seed)
    ring = ctxs[0].ring
    kseed = np.random.SeedSequence([0xB200_4B45, B.key_seed()]).generate_state(8, dtype=np.uint32)
    spec = (ring.log_n, ring.t, ring.L, ring.n_slots, ring.one_row, ring.q_bits)

    # the oracle side starts from the same ciphertext words, encryption streams and channel seeds
    from dataclasses import replace

    inputs = []
    for h in range(H):
        segs = {name: (seg, [(pt.words(), pt.noise_budget) for pt in seg.parts]) for name, seg in caches[h].segments()}
        inputs.append((segs, (qs[h].words(), qs[h].noise_budget), ctxs[h]._enc_key.copy(), ctxs[h]._enc_index))

    def oracle_head(h):
        segs, (qw, qb), key, idx = inputs[h]
        o = oracle_mod.OracleRing(*spec[:5], kseed, q_bits=spec[5])
        oc = OracleContext(ctxs[h].params, o, key, idx)
        conv = {name: api.PackedMatrix(seg.encoding, [oc.wrap(w, b) for w, b in parts], encrypted=True,
                                       slot_period=seg.slot_period) for name, (seg, parts) in segs.items()}
        ocache = replace(caches[h], **conv)
        ch = api.MpcChannel(p, seed=seed + 100 + h)
        out = ref.attention_step(oc.wrap(qw, qb), ocache, fp, oc, ch)
        return out, oc.counter.as_dict(), ch.transcript

    with cf.ThreadPoolExecutor(H) as ex:
        futs = [ex.submit(oracle_head, h) for h in range(H)]
        snaps = [c.counter.snapshot() for c in ctxs]
        res = api.attention_step_heads(qs, caches, fp, ctxs, chans)
        want = [f.result() for f in futs]
    for h in range(H):
        out, counts, transcript = want[h]
        assert np.array_equal(res[h].words(), out.words()), f"head {h}: output ciphertext words differ"
        assert ctxs[h].counter.delta(snaps[h]) == counts, h
        assert chans[h].transcript == transcript, h
        assert res[h].noise_budget == out.noise_budget
        assert np.array_equal(ctxs[h].decrypt(res[h]), oracle_mod.OracleRing(*spec[:5], kseed, q_bits=spec[5])
                              .decrypt(out.words()))


def test_prefill_words_equal_reference_sequence(oracle_mod):
    """Encrypted prefill attention (2 heads, n = 8192, m = 3, d2 = 2) on the
    production ring: the head-batched B200 sweep against the reference's op
    sequence (arcc.py:248-317) executed op by op on the CPU RNS-BFV oracle --
    every output ciphertext word, counter and transcript entry."""
    from dataclasses import replace  # noqa: F401

    import harness
    from hostapi import repo_api
    from oracle import reference_path as ref
    from oracle.rns_context import OracleContext
    from paper_2602_08798_b200 import backend as B
    from paper_2602_08798_b200._native import build

    build()
    api = repo_api()
    n, p, m, d2, H = 8192, harness.P8192, 3, 2, 2
    params = api.BackendParams(n_slots=n, plain_modulus=p)
    root = B.GpuContext(params, 31)
    fp = api.FixedPointParams(8, p)
    rng = np.random.default_rng(31)
    ctxs = [root.fork() for _ in range(H)]
    mats = [[api.encode(np.mod(api.fp_encode(rng.uniform(-1, 1, (m, d2)), fp), p), api.EncodingKind.OUTER, c)
             for _ in range(3)] for c in ctxs]
    ring = ctxs[0].ring
    kseed = np.random.SeedSequence([0xB200_4B45, B.key_seed()]).generate_state(8, dtype=np.uint32)
    spec = (ring.log_n, ring.t, ring.L, ring.n_slots, ring.one_row, ring.q_bits)
    inputs = [([[(pt.words(), pt.noise_budget) for pt in P.parts] for P in mats[h]], ctxs[h]._enc_key.copy(),
               ctxs[h]._enc_index) for h in range(H)]

    def oracle_head(h):
        parts, key, idx = inputs[h]
        oc = OracleContext(params, oracle_mod.OracleRing(*spec[:5], kseed, q_bits=spec[5]), key, idx)
        Q, K, V = (api.PackedMatrix(mats[h][k].encoding, [oc.wrap(w, b) for w, b in parts[k]], encrypted=True)
                   for k in range(3))
        ch = api.MpcChannel(p, seed=70 + h)
        out = ref.prefill_attention(Q, K, V, fp, oc, ch)
        return out, oc.counter.as_dict(), ch.transcript

    chans = [api.MpcChannel(p, seed=70 + h) for h in range(H)]
    with cf.ThreadPoolExecutor(H) as ex:
        futs = [ex.submit(oracle_head, h) for h in range(H)]
        snaps = [c.counter.snapshot() for c in ctxs]
        res = api.prefill_attention_heads([x[0] for x in mats], [x[1] for x in mats], [x[2] for x in mats], fp, ctxs,
                                          chans)
        want = [f.result() for f in futs]
    for h in range(H):
        out, counts, transcript = want[h]
        for a, b in zip(res[h].parts, out.parts):
            assert np.array_equal(a.words(), b.words()), f"head {h}: output words differ"
            assert a.noise_budget == b.noise_budget
        assert ctxs[h].counter.delta(snaps[h]) == counts
        assert chans[h].transcript == transcript


def test_batched_mult_cipher_both_resident_bitexact(bench):
    """16 a-operands each multiplied by 16 b's (the decode step's a_pref x V
    columns pattern) with BOTH base-B extensions resident (cgb_mult_cipher_ext2,
    the path w_mult_cipher takes when a repeats): the oracle's words."""
    g, pool, vals, ids, words = bench
    ai = np.repeat(np.arange(16), 16)
    bi = (np.arange(256) * 7 + 3) % COUNT
    out = g.alloc(256)
    g.mult_cipher_ext2(ids[ai], g.ext_B(ids[ai]), ids[bi], g.ext_B(ids[bi]), out)
    got = g.store(out)
    want = pool.map(lambda o, i, j: o.mult_cipher(words[i], words[j]), ai, bi)
    bad = [i for i in range(256) if not np.array_equal(got[i], want[i])]
    assert not bad, f"{len(bad)} items differ, first {bad[:8]}"
    g.free(out)


def test_reencrypt_equals_decrypt_then_encrypt(bench):
    """The client's re-encryption of a refresh on the device (cgb_reencrypt_batch)
    == decrypt to host slots, then encrypt them (kv_cache.py:150): every word."""
    g, pool, vals, ids, words = bench
    src = ids[:16]
    keys = np.stack([ENC + 7 * i for i in range(16)]).astype(np.uint32)
    idx = np.arange(100, 116, dtype=np.uint64)
    a = g.alloc(16)
    g.reencrypt_batch(src, keys, idx, a)
    b = g.alloc(16)
    g.encrypt_batch(g.decrypt(src), keys, idx, b)
    assert np.array_equal(g.store(a), g.store(b))
    assert np.array_equal(g.decrypt(a), vals[:16])
    g.free(np.concatenate([a, b]))
