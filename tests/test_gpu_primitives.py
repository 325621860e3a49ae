"""GPU primitives vs the CPU RNS-BFV oracle: every ciphertext word bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KEY = np.arange(8, dtype=np.uint32) * 7 + 1
ENC = np.arange(8, dtype=np.uint32) + 1000

CASES = [
    # (log_n, t, L, n_slots, one_row, q_bits)
    (4, 97, 3, 8, True, 60),
    (3, 17, 2, 8, False, 60),
    (7, 67109633, 4, 64, True, 60),
    (14, 536903681, 4, 8192, True, 60),   # integer-pipe NTT
    (14, 536903681, 4, 8192, True, 49),   # FP64-pipe NTT
    (13, 536903681, 3, 4096, True, 49),
    (14, 536903681, 3, 8192, True, 49),   # the benchmarked ring (bench.py decode step)
    (14, 536903681, 2, 8192, True, 49),
    (15, 537133057, 4, 16384, True, 49),  # config 5: N = 2^15 (p = 1 mod 2^16)
    (16, 537133057, 3, 32768, True, 49),  # config 5: N = 2^16 (p = 1 mod 2^17)
    (13, 536903681, 8, 4096, True, 49),   # config 5: 8 primes
    (14, 536903681, 6, 8192, True, 49),   # config 5: fused key switch with > 4 digits
    (16, 537133057, 8, 32768, True, 49),  # config 5: the widest ring
]


@pytest.fixture(scope="module", params=CASES,
                ids=lambda c: f"logN{c[0]}_t{c[1]}_L{c[2]}_{'row' if c[4] else 'two'}_q{c[5]}")
def pair(request, oracle_mod):
    from paper_2602_08798_b200._native import build
    from paper_2602_08798_b200.ring import Ring

    build()
    log_n, t, L, n, one_row, qb = request.param
    g = Ring(log_n, t, L, n, one_row, KEY, arena_cts=64, arena_pts=16, q_bits=qb)
    o = oracle_mod.OracleRing(log_n, t, L, n, one_row, KEY, q_bits=qb)
    return g, o


def test_moduli_match(pair):
    g, o = pair
    assert g.moduli == o.moduli[: len(g.moduli)]


def _enc(g, o, v, idx):
    ids = g.alloc(1)
    g.encrypt(v, ENC, idx, ids)
    ref = o.encrypt(v, ENC, idx)
    return ids, ref


def test_encrypt_decrypt_bitexact(pair, rng):
    g, o = pair
    v = rng.integers(0, o.t, o.n_slots)
    ids, ref = _enc(g, o, v, 5)
    assert np.array_equal(g.store(ids)[0], ref)
    assert np.array_equal(g.decrypt(ids)[0], v)


def test_pointwise_ops_bitexact(pair, rng):
    g, o = pair
    v, w = rng.integers(0, o.t, (2, o.n_slots))
    a, ra = _enc(g, o, v, 1)
    b, rb = _enc(g, o, w, 2)
    out = g.alloc(1)
    g.add(a, b, out)
    assert np.array_equal(g.store(out)[0], o.add(ra, rb))
    pt = g.alloc_pt(2)
    g.encode_pt(w, 1, pt[:1])
    g.add_plain(a, pt[:1], out)
    assert np.array_equal(g.store(out)[0], o.add_plain(ra, w))
    g.encode_pt(w, 0, pt[1:])
    g.mult_plain(a, pt[1:], out)
    assert np.array_equal(g.store(out)[0], o.mult_plain(ra, w))
    assert np.array_equal(g.decrypt(out)[0], (v * w) % o.t)


def test_rotate_bitexact(pair, rng):
    g, o = pair
    v = rng.integers(0, o.t, o.n_slots)
    a, ra = _enc(g, o, v, 3)
    out = g.alloc(1)
    h = o.n_slots if o.one_row else o.n_slots // 2
    for k in [0, 1, 3, h - 1]:
        gel = pow(5, k % h, 2 * o.N)
        g.galois(a, gel, out)
        assert np.array_equal(g.store(out)[0], o.galois(ra, gel)), k
        if o.one_row:
            assert np.array_equal(g.decrypt(out)[0], np.roll(v, -k))


def test_rotate_hoisted_bitexact(pair, rng):
    """A wave of rotations of ONE source (the CPVM's diagonal steps) takes the
    hoisted key switch (one ModUp, per-step gathers): same words as the oracle,
    with and without the fused add of the input."""
    g, o = pair
    if not o.one_row:
        pytest.skip("cgb_rotate needs the one-row layout")
    v = rng.integers(0, o.t, o.n_slots)
    a, ra = _enc(g, o, v, 4)
    steps = np.array([1, 2, 5, o.n_slots - 1, 7, 3], np.int64)
    src = np.repeat(a, steps.size)
    for add in (False, True):
        out = g.alloc(steps.size)
        g.rotate(src, steps, out, add_input=add)
        got = g.store(out)
        for i, k in enumerate(steps):
            want = o.galois(ra, pow(5, int(k) % o.n_slots, 2 * o.N))
            if add:
                want = o.add(want, ra)
            assert np.array_equal(got[i], want), (add, k)
        g.free(out)


def test_mult_cipher_bitexact(pair, rng):
    g, o = pair
    v, w = rng.integers(0, o.t, (2, o.n_slots))
    a, ra = _enc(g, o, v, 7)
    b, rb = _enc(g, o, w, 8)
    out = g.alloc(1)
    g.mult_cipher(a, b, out)
    ref = o.mult_cipher(ra, rb)
    assert np.array_equal(g.store(out)[0], ref)
    assert np.array_equal(g.decrypt(out)[0], (v * w) % o.t)


def test_mult_cipher_resident_extension_bitexact(pair, rng):
    """mult_cipher with b's base-B extension kept resident: the same words as
    mult_cipher, the extension reused across calls and freed with b."""
    g, o = pair
    v, w = rng.integers(0, o.t, (2, o.n_slots))
    a, ra = _enc(g, o, v, 11)
    b, rb = _enc(g, o, w, 12)
    ref = o.mult_cipher(ra, rb)
    out = g.alloc(2)
    bb = np.concatenate([b, b])
    g.mult_cipher_ext(np.concatenate([a, a]), bb, g.ext_B(bb), out)
    words = g.store(out)
    assert np.array_equal(words[0], ref) and np.array_equal(words[1], ref)
    assert int(b[0]) in g._ext
    g.free(b)
    assert int(b[0]) not in g._ext
    g.free(np.concatenate([a, out]))


def test_rings_of_different_sizes_coexist():
    """Kernel attributes are process-global: a smaller ring created later must not
    break a larger one created earlier (regression)."""
    from paper_2602_08798_b200.ring import Ring

    big = Ring(5, 193, 3, 16, True, KEY, arena_cts=8, arena_pts=4)
    small = Ring(3, 17, 2, 4, True, KEY, arena_cts=8, arena_pts=4)
    for r in (big, small, big):
        ids = r.alloc(1)
        v = np.arange(r.n_slots) % r.t
        r.encrypt(v, ENC, 0, ids)
        assert np.array_equal(r.decrypt(ids)[0], v)
        r.free(ids)
