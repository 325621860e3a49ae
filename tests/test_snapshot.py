"""KV-cache checkpoints: the reference's decrypted snapshot
(/root/reference/pkg/src/cryptogen/kv_cache.py:219-281, its test
tests/test_kv_cache.py:246-266) and the ciphertext-level snapshot
(save_cache_ct / load_cache_ct: raw RNS words, no client)."""
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
import harness  # noqa: E402
from hostapi import repo_api  # noqa: E402


def _cache(api, ctx, rng, fp, p, d2=4):
    tok = lambda: np.mod(api.fp_encode(rng.uniform(-1, 1, d2), fp), p)  # noqa: E731
    Kp = api.encode(np.mod(api.fp_encode(rng.uniform(-1, 1, (2, d2)), fp), p), api.EncodingKind.OUTER, ctx)
    Vp = api.encode(np.mod(api.fp_encode(rng.uniform(-1, 1, (2, d2)), fp), p), api.EncodingKind.OUTER, ctx)
    cache = api.init_cache(Kp, Vp, ctx)
    for _ in range(3):
        kv = tok()
        cache = api.append_token(cache, api.pack_token_inner(kv, ctx), api.pack_token_inner(kv, ctx), ctx)
    return cache, tok


def _roundtrip_slots(api, new_ctx, tmp_path):
    p = harness.P64
    fp = api.FixedPointParams(8, p)
    ctx = new_ctx(api.BackendParams(n_slots=64, plain_modulus=p), 0)
    rng = np.random.default_rng(0)
    cache, tok = _cache(api, ctx, rng, fp, p)
    api.save_cache(cache, tmp_path / "snap", ctx)
    loaded = api.load_cache(tmp_path / "snap", ctx)
    assert api.cache_stats(loaded) == api.cache_stats(cache)
    q = api.pack_token_inner(tok(), ctx)
    a = ctx.decrypt(api.attention_step(q, cache, fp, ctx, api.MpcChannel(p, seed=5)))
    b = ctx.decrypt(api.attention_step(q, loaded, fp, ctx, api.MpcChannel(p, seed=6)))
    assert (a == b).all()
    for (_, s0), (_, s1) in zip(cache.segments(), loaded.segments()):
        assert [pt.noise_budget for pt in s0.parts] == [pt.noise_budget for pt in s1.parts]


def test_slots_snapshot_roundtrip_slot_oracle(tmp_path):
    from oracle.slots import SlotContext

    _roundtrip_slots(repo_api(), SlotContext, tmp_path)


@pytest.mark.gpu
def test_slots_snapshot_roundtrip_gpu(tmp_path):
    from paper_2602_08798_b200._native import build
    from paper_2602_08798_b200.backend import GpuContext

    build()
    _roundtrip_slots(repo_api(), GpuContext, tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("n,p", [(64, harness.P64), (8192, harness.P8192)])
def test_ciphertext_snapshot_roundtrip_gpu(tmp_path, n, p):
    """Equal words, budgets and ids after save_cache_ct -> load_cache_ct, and the
    same attention output; a snapshot of another ring is rejected."""
    from paper_2602_08798_b200._native import build
    from paper_2602_08798_b200.backend import GpuContext, ParameterError

    build()
    api = repo_api()
    fp = api.FixedPointParams(8, p)
    ctx = GpuContext(api.BackendParams(n_slots=n, plain_modulus=p), 0)
    cache, tok = _cache(api, ctx, np.random.default_rng(1), fp, p)
    api.save_cache_ct(cache, tmp_path / "ct", ctx)
    snap = ctx.counter.snapshot()
    loaded = api.load_cache_ct(tmp_path / "ct", ctx)
    assert ctx.counter.delta(snap) == {k: 0 for k in snap.as_dict()}  # loading is not an HE op
    assert api.cache_stats(loaded) == api.cache_stats(cache)
    for (n0, s0), (n1, s1) in zip(cache.segments(), loaded.segments()):
        assert n0 == n1 and s0.encoding == s1.encoding and s0.slot_period == s1.slot_period
        for a, b in zip(s0.parts, s1.parts):
            assert np.array_equal(a.words(), b.words())
            assert (a.noise_budget, a.id) == (b.noise_budget, b.id)
    q = api.pack_token_inner(tok(), ctx)
    o1 = api.attention_step(q, cache, fp, ctx, api.MpcChannel(p, seed=5))
    o2 = api.attention_step(q, loaded, fp, ctx, api.MpcChannel(p, seed=5))
    assert np.array_equal(ctx.decrypt(o1), ctx.decrypt(o2))
    # load_cache reads both formats; a snapshot of another ring (other moduli) is rejected
    assert api.cache_stats(api.load_cache(tmp_path / "ct", ctx)) == api.cache_stats(cache)
    import json
    import shutil

    shutil.copytree(tmp_path / "ct", tmp_path / "other")
    man = json.loads((tmp_path / "other" / "manifest.json").read_text())
    man["ring"]["moduli"][0] += 2
    (tmp_path / "other" / "manifest.json").write_text(json.dumps(man))
    with pytest.raises(ParameterError):
        api.load_cache_ct(tmp_path / "other", ctx)
    api.save_cache(cache, tmp_path / "slots", ctx)
    with pytest.raises(ParameterError):
        api.load_cache_ct(tmp_path / "slots", ctx)
