"""Host code of the hot path over the slot oracle vs golden vectors recorded
from the reference (tests/golden/make_golden.py).  CPU only."""
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
import harness  # noqa: E402
from hostapi import compare, repo_api  # noqa: E402

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def api():
    return repo_api()


def slot_ctx(params, seed):
    from oracle.slots import SlotContext

    return SlotContext(params, seed)


@pytest.mark.parametrize("name", list(harness.SMALL))
def test_small_scenarios_match_reference(api, name):
    fn, kw = harness.SMALL[name]
    rec, _ = fn(api, slot_ctx, **kw)
    compare(rec, np.load(GOLD / f"{name}.npz"))


@pytest.mark.parametrize("name", ["full_attn_m128", "full_attn_m96_t32", "full_attn_m0_t130"])
def test_full_size_decode_matches_reference(api, name):
    fn, kw = harness.FULL[name]
    rec, _ = fn(api, slot_ctx, **kw)
    compare(rec, np.load(GOLD / f"{name}.npz"))


def test_full_size_prefill_matches_reference(api):
    fn, kw = harness.FULL["full_prefill_m128"]
    rec, _ = fn(api, slot_ctx, **kw)
    compare(rec, np.load(GOLD / "full_prefill_m128.npz"))


def test_reference_path_restatement_matches_goldens(api):
    """oracle/reference_path.py (the sequential per-op restatement used as the
    CPU baseline and as the per-op GPU path) reproduces the reference."""
    from types import SimpleNamespace

    from oracle import reference_path as ref

    ns = SimpleNamespace(**vars(api))
    ns.attention_step, ns.append_token, ns.maybe_refresh = ref.attention_step, ref.append_token, ref.maybe_refresh
    for name in ("attn_m5_t19", "attn_m16_t40_refresh"):
        fn, kw = harness.SMALL[name]
        rec, _ = fn(ns, slot_ctx, **kw)
        compare(rec, np.load(GOLD / f"{name}.npz"))


def test_softmax_rows_equals_per_row():
    """The head-batched integer softmax (fixedpoint.attention_weights_rows) equals
    the per-row restatement of fixedpoint.py:204-209 on random score ranges."""
    from paper_2602_08798_b200.fixedpoint import FixedPointParams, attention_weights, attention_weights_rows
    p = 536903681
    rng = np.random.default_rng(7)
    for f in (6, 8, 11):
        fp = FixedPointParams(f, p)
        for n in (2, 17, 129, 513):
            for scale in (1, 2 ** f, 2 ** (2 * f + 6)):
                S = rng.integers(-4 * scale, 4 * scale, (12, n))
                ref = np.stack([attention_weights(S[h], 64, fp) for h in range(12)])
                assert (attention_weights_rows(S, 64, fp) == ref).all()


@pytest.mark.parametrize("groups", [2, 3])
def test_interleaved_head_groups_equal_one_schedule(api, groups):
    """attention_step_heads with the heads as interleaved groups (one group's client
    round trip overlapping the next group's device work) charges and returns exactly
    what the single schedule does: outputs, ids, budgets, counters, transcripts."""
    from paper_2602_08798_b200 import arcc

    def run(g):
        root, fp, ctxs, caches, qs, chans = harness.attention_heads(api, slot_ctx, 64, harness.P64, 4, 6, 5, 6,
                                                                    seed=3)
        outs = arcc.attention_step_heads(qs, caches, fp, ctxs, chans, groups=g)
        return ([np.asarray(o.slots).tolist() for o in outs], [o.id % harness.ID_BASE for o in outs], [o.noise_budget for o in outs],
                [c.counter.as_dict() for c in ctxs], [ch.transcript for ch in chans],
                [ch.sample_mask(4).tolist() for ch in chans])

    assert run(1) == run(groups)


def test_wave_content_classes():
    """Wave bookkeeping behind the rotation dedup: repeated handles share a class,
    take() keeps classes, concat() gives class-less waves fresh distinct classes."""
    from paper_2602_08798_b200.backend import Wave

    aids = np.array([7, 7, 9], np.uint32)
    w = Wave([None], np.zeros(3, np.int64), aids, np.zeros(3, np.int64), [], klass=-(aids.astype(np.int64) + 1))
    t = w.take([2, 0, 1, 0])
    assert t.klass.tolist() == [-10, -8, -8, -8]
    plain = Wave([None], np.zeros(2, np.int64), np.array([1, 2], np.uint32), np.zeros(2, np.int64), [])
    c = Wave.concat([t, plain])
    assert c.klass[:4].tolist() == t.klass.tolist()
    assert c.klass[4] != c.klass[5] and min(c.klass[4:]) > 0
    assert Wave.concat([plain, plain]).klass is None


def _prefill_heads(api, new_ctx, n, p, m, d2, H, batched, seed=3):
    params = api.BackendParams(n_slots=n, plain_modulus=p)
    root = new_ctx(params, seed)
    fp = api.FixedPointParams(8, p)
    rng = np.random.default_rng(seed)
    ctxs = [root.fork() for _ in range(H)]
    mats = [[api.encode(np.mod(api.fp_encode(rng.uniform(-1, 1, (m, d2)), fp), p), api.EncodingKind.OUTER, c)
             for _ in range(3)] for c in ctxs]
    chans = [api.MpcChannel(p, seed=50 + h) for h in range(H)]
    if batched:
        outs = api.prefill_attention_heads([x[0] for x in mats], [x[1] for x in mats], [x[2] for x in mats], fp, ctxs,
                                           chans)
    else:
        outs = [api.prefill_attention(x[0], x[1], x[2], fp, c, ch) for x, c, ch in zip(mats, ctxs, chans)]
    return outs, ctxs, chans


def test_prefill_heads_batched_equals_per_head(api):
    """prefill_attention_heads (all heads swept together: one key per shift for
    every head's columns) == one prefill_attention per head: outputs, budgets,
    counters, transcripts, next masks (arcc.py:248-317)."""
    from oracle.slots import SlotContext

    res = {}
    for batched in (False, True):
        outs, ctxs, chans = _prefill_heads(api, SlotContext, 64, harness.P64, 5, 4, 3, batched)
        res[batched] = ([api.decode(o, c).tolist() for o, c in zip(outs, ctxs)],
                        [[pt.noise_budget for pt in o.parts] for o in outs],
                        [c.counter.as_dict() for c in ctxs], [ch.transcript for ch in chans],
                        [ch.sample_mask(4).tolist() for ch in chans])
    assert res[False] == res[True]
