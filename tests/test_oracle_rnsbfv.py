"""Pin the CPU RNS-BFV restatement: textbook known-answer properties, and
decrypt(op(encrypt(v))) == the reference's slot semantics (backend.py:307-355)."""
import numpy as np
import pytest

KEY = np.arange(8, dtype=np.uint32)
ENC = np.arange(8, dtype=np.uint32) + 100


@pytest.fixture(scope="module")
def small(oracle_mod):
    return oracle_mod.OracleRing(4, 97, 3, 8, True, KEY)


def brev(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2)


def test_ntt_is_negacyclic_convolution(small, rng):
    N, q = small.N, small.moduli[0]
    a, b = rng.integers(0, q, (2, N), dtype=np.uint64)
    c = small.intt(0, np.array([int(x) * int(y) % q for x, y in zip(small.ntt(0, a), small.ntt(0, b))],
                                dtype=np.uint64))
    ref = [0] * N
    for i in range(N):
        for j in range(N):
            v = int(a[i]) * int(b[j])
            ref[(i + j) % N] += -v if i + j >= N else v
    assert [int(x) for x in c] == [x % q for x in ref]
    assert np.array_equal(small.intt(0, small.ntt(0, a)), a)


def test_ntt_evaluation_order(small, rng):
    N, q = small.N, small.moduli[0]
    a = rng.integers(0, q, N, dtype=np.uint64)
    A = small.ntt(0, a)
    psi = next(p for p in (pow(x, (q - 1) // (2 * N), q) for x in range(2, 200)) if pow(p, N, q) == q - 1)
    for k in range(N):
        e = 2 * brev(k, small.log_n) + 1
        assert int(A[k]) == sum(int(a[i]) * pow(psi, e * i, q) for i in range(N)) % q


def test_primes_and_chain(oracle_mod):
    o = oracle_mod.OracleRing(14, 536903681, 4, 8192, True, KEY)
    assert [m.bit_length() for m in o.moduli] == [60] * 4 + [61] * 6
    assert all(m % (2 * o.N) == 1 for m in o.moduli)
    assert len(set(o.moduli)) == len(o.moduli)


def test_slot_semantics(small, rng):
    t, n = small.t, small.n_slots
    v, w = rng.integers(0, t, (2, n))
    a, b = small.encrypt(v, ENC, 0), small.encrypt(w, ENC, 1)
    assert np.array_equal(small.decrypt(a), v)
    assert np.array_equal(small.decrypt(small.add(a, b)), (v + w) % t)
    assert np.array_equal(small.decrypt(small.add_plain(a, w)), (v + w) % t)
    assert np.array_equal(small.decrypt(small.mult_plain(a, w)), (v * w) % t)
    assert np.array_equal(small.decrypt(small.mult_cipher(a, b)), (v * w) % t)
    for k in range(n):
        assert np.array_equal(small.decrypt(small.rotate(a, k)), np.roll(v, -k))


def test_reference_examples(oracle_mod):
    """tests/test_backend.py:98-110 of the reference: rotate [1,2,3,4] by 1."""
    o = oracle_mod.OracleRing(3, 17, 2, 4, True, KEY)
    ct = o.encrypt([1, 2, 3, 4], ENC, 0)
    assert o.decrypt(o.rotate(ct, 1)).tolist() == [2, 3, 4, 1]
    assert o.decrypt(o.rotate(ct, 0)).tolist() == [1, 2, 3, 4]


def test_noise_budget_tracks_ledger_scale(oracle_mod, rng):
    o = oracle_mod.OracleRing(14, 536903681, 4, 8192, True, KEY)
    v = rng.integers(0, o.t, o.n_slots)
    ct = o.encrypt(v, ENC, 0)
    fresh = o.noise_budget(ct)
    assert fresh > 190
    mc = o.mult_cipher(ct, o.encrypt(v, ENC, 1))
    assert 30 < fresh - o.noise_budget(mc) < 60
    assert fresh - o.noise_budget(o.rotate(ct, 5)) < 10
