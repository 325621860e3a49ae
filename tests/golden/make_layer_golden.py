"""Record the decoder-layer golden (BASELINE config 3 shape, toy size) from the
REFERENCE's own encrypted pipeline.

Run here (the reference is importable only in this container):
    python tests/golden/make_layer_golden.py
Imports cryptogen from /root/reference/pkg/src, builds the reference's toy
model (model.py:95-99 config, generate_toy_model weights), runs its
``prefill`` and ``decode_step`` (model.py:425-566) on the slot emulation with
every cache part force-refreshed before each step (config 3's "noise refresh
each step", kv_cache.py:156 force=True), and writes tests/golden/layer_toy.npz:
weights, prompt, generated tokens, every step's logits, op counters, MPC
byte totals, every channel's transcript and its next mask draws.  /root/reference is never read at test time.
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

# name -> (n_slots, plain modulus, model config or None for the toy config, prompt, steps)
CASES = {
    "layer_toy": (64, 67109633, None, [5, 17, 3, 60, 22, 9], 3),  # harness.P64
    # the production ring (n = 8192, p = 536903681 -> N = 16384, FP64-pipe kernels)
    "layer_n8192": (8192, 536903681, dict(layers=1, d1=128, heads=2, ffn_dim=256, vocab=512, max_seq=64, f=8),
                    [7, 300, 41, 511, 2, 96, 180, 33], 2),
}


def main():
    for name, case in CASES.items():
        record(name, *case)


def record(name, N, P, cfg_kw, PROMPT, STEPS):
    from cryptogen import backend, kv_cache, model as M

    cfg = M.toy_config() if cfg_kw is None else M.ModelConfig(**cfg_kw)
    mdl = M.generate_toy_model(cfg, seed=0)
    ctx = backend.new_context(backend.BackendParams(n_slots=N, plain_modulus=P), 0)
    chans = M._channels(0, cfg.layers, cfg.heads, P)
    state = M.prefill(mdl, PROMPT, ctx, chans)
    logits = [state.next_logits.astype(np.int64)]
    tokens = []
    for _ in range(STEPS):
        state.caches = [[kv_cache.maybe_refresh(state.caches[l][h], ctx, chans[(l, h)], force=True)
                         for h in range(cfg.heads)] for l in range(cfg.layers)]
        tok, state = M.decode_step(mdl, state, ctx, chans)
        tokens.append(tok)
        logits.append(state.next_logits.astype(np.int64))
    oracle = M.oracle_generate(mdl, PROMPT, STEPS, P)
    assert oracle == tokens, (oracle, tokens)
    rec = {f"w_{k}": v for k, v in mdl.weights.items()}
    rec.update(config=json.dumps(cfg.as_dict()), prompt=np.array(PROMPT), tokens=np.array(tokens),
               logits=np.stack(logits), counters=json.dumps(ctx.counter.as_dict(), sort_keys=True),
               mpc_bytes=np.int64(sum(ch.bytes_sent for ch in chans.values())), n=N, p=P,
               transcripts=json.dumps({str(k): ch.transcript for k, ch in chans.items()}, sort_keys=True),
               next_masks=json.dumps({str(k): ch.sample_mask(4).tolist() for k, ch in chans.items()}, sort_keys=True))
    np.savez_compressed(HERE / f"{name}.npz", **rec)
    print(name, "tokens", tokens, "counters", ctx.counter.as_dict())


if __name__ == "__main__":
    main()
