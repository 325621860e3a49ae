"""Decoder-layer pipeline (paper_2602_08798_b200.model, BASELINE config 3) vs the
reference's own encrypted pipeline: goldens recorded by
tests/golden/make_layer_golden.py -- the reference's toy model (2 layers, 4
heads, n = 64, prompt 6, 3 greedy steps) and a 1-layer model (d1 128, 2 heads,
d_ff 256, vocab 512) on the production ring n = 8192 (prompt 8, 2 steps), every
cache part force-refreshed before each step.
Tokens, every step's logits, op counters, MPC byte totals, every channel's
transcript and next mask draws must be equal."""
import json
from pathlib import Path

import numpy as np
import pytest

from conftest import gpu_available

GOLDS = Path(__file__).resolve().parent / "golden"
CASES = ["layer_toy", "layer_n8192"]  # n = 64 toy model; 1 layer on the production ring (n = 8192)


def _run(make_ctx, case="layer_toy"):
    from paper_2602_08798_b200 import model as M
    from paper_2602_08798_b200.backend import BackendParams

    g = np.load(GOLDS / f"{case}.npz")
    cfg = M.ModelConfig(**json.loads(str(g["config"])))
    mdl = M.Model(cfg, {k[2:]: g[k] for k in g.files if k.startswith("w_")})
    p = int(g["p"])
    ctx = make_ctx(BackendParams(n_slots=int(g["n"]), plain_modulus=p), 0)
    chans = M.channels(0, cfg.layers, cfg.heads, p)
    state = M.prefill(mdl, [int(t) for t in g["prompt"]], ctx, chans)
    logits, toks = [state.next_logits], []
    for _ in range(len(g["tokens"])):
        tok, state = M.decode_step(mdl, state, ctx, chans, force_refresh=True)
        toks.append(tok)
        logits.append(state.next_logits)
    assert toks == [int(t) for t in g["tokens"]]
    assert np.array_equal(np.stack(logits), g["logits"])
    assert ctx.counter.as_dict() == json.loads(str(g["counters"]))
    assert sum(ch.bytes_sent for ch in chans.values()) == int(g["mpc_bytes"])
    # every channel's transcript in the reference's order, and its generator at the same
    # point of its stream (the masks, hence every share, were drawn in the same order)
    assert json.dumps({str(k): ch.transcript for k, ch in chans.items()}, sort_keys=True) == str(g["transcripts"])
    assert json.dumps({str(k): ch.sample_mask(4).tolist() for k, ch in chans.items()},
                      sort_keys=True) == str(g["next_masks"])
    return ctx, state


@pytest.mark.parametrize("case", CASES)
def test_layer_pipeline_on_slot_oracle(case):
    from oracle.slots import SlotContext

    _run(SlotContext, case)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_layer_pipeline_on_gpu(case):
    assert gpu_available()
    from paper_2602_08798_b200._native import build
    from paper_2602_08798_b200.backend import GpuContext

    build()
    ctx, state = _run(GpuContext, case)
    assert all(c.noise_budget > 0 for cache in state.caches[0] for c in cache.prefill_K.parts)


def test_cpmm_chunked_equals_unchunked():
    """Wide CPMM outputs are computed in column chunks: same decrypted columns."""
    from oracle.slots import SlotContext
    from paper_2602_08798_b200 import linear_kernels as LK
    from paper_2602_08798_b200.backend import BackendParams
    from paper_2602_08798_b200.encodings import EncodingKind, decode, encode

    p = 67109633
    ctx = SlotContext(BackendParams(n_slots=64, plain_modulus=p), 0)
    rng = np.random.default_rng(3)
    X = encode(rng.integers(0, 50, (8, 24)), EncodingKind.OUTER, ctx)
    W = encode(rng.integers(-30, 30, (24, 40)), EncodingKind.DIAGONAL, ctx, encrypted=False)
    full = decode(LK.cpmm_outer_diagonal(X, W, ctx), ctx)
    old = LK.CPMM_CHUNK
    try:
        LK.CPMM_CHUNK = 7
        chunked = decode(LK.cpmm_outer_diagonal(X, W, ctx), ctx)
    finally:
        LK.CPMM_CHUNK = old
    assert np.array_equal(full, chunked)


def _wide_vocab_logits(make_ctx):
    """Unembedding wider than the slot count (vocab 200 at n = 64: 4 blocks)
    equals the plain fixed-point product x W, truncated."""
    from paper_2602_08798_b200 import model as M
    from paper_2602_08798_b200.backend import BackendParams
    from paper_2602_08798_b200.fixedpoint import fp_truncate, to_signed

    g = np.load(GOLDS / "layer_toy.npz")
    p, n = int(g["p"]), int(g["n"])
    cfg = M.ModelConfig(layers=1, d1=32, heads=4, ffn_dim=64, vocab=200, max_seq=8, f=8)
    mdl = M.gpt2_layer_model(cfg, seed=3)
    ctx = make_ctx(BackendParams(n_slots=n, plain_modulus=p), 0)
    fp = mdl.fixed_point(ctx)
    x = np.random.default_rng(1).integers(-300, 300, cfg.d1)
    xv = np.zeros(n, np.int64)
    xv[:cfg.d1] = np.mod(x, p)
    x_ct = ctx.encrypt(ctx.plain_from_dense(xv))
    got = M._logits(mdl, x_ct, ctx, fp)
    want = fp_truncate(to_signed(np.mod(x @ mdl.unembed(), p), p), fp.f)
    assert got.shape == (200,)
    assert np.array_equal(got, want)
    assert ctx.counter.rotate > 0


def test_wide_vocab_unembedding_on_slot_oracle():
    from oracle.slots import SlotContext

    _wide_vocab_logits(SlotContext)


@pytest.mark.gpu
def test_wide_vocab_unembedding_on_gpu():
    assert gpu_available()
    from paper_2602_08798_b200._native import build
    from paper_2602_08798_b200.backend import GpuContext

    build()
    _wide_vocab_logits(GpuContext)
