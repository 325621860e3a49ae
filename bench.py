"""Encrypted-KV attention decode on one B200: ms/token (BASELINE.json metric).

Workload ("decode_attention_12h_L{L}"): one decode token of a GPT-2-small
attention layer under RNS-BFV -- 12 heads, d_head = 64, n = 8192 slots,
p = 536903681 (the reference's default parameter set), a cached prefill of
L tokens per head (outer-packed K/V), then per step:
lazy refresh check, append of the new K/V token into the compacted
generated segment, and the heterogeneous attention step of all 12 heads
(arcc.attention_step_heads).  Synthetic fixed-point inputs, uniform in
[-1, 1] at f = 8, seeded.

value: device-resident step (encrypted q/k/v tokens already in HBM).
e2e:   same step through the public API from HOST plaintext tokens: client
       encryption of q/k/v (H2D) ... decryption of the 12 head outputs (D2H).
Both include the MPC client round trips of the attention step itself
(masked decrypts / re-encryptions), which are part of the reference path.

--impl reference: the reference's CPU path (sequential per-op restatement
of the emulation, oracle/reference_path.py over oracle/slots.py) on the
same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("CGB_KEY_SEED", "0")  # a reproducible keyring for the measurement

P = 536903681
N_SLOTS = 8192
D2 = 64
HEADS = 12
F = 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="decode", choices=["decode", "prefill", "layer"])
    ap.add_argument("--L", type=int, default=128, help="cached prefill length per head")
    ap.add_argument("--heads", type=int, default=HEADS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--full-vocab", action="store_true",
                    help="layer workload: unembed all 50257 columns (7 slot blocks) instead of the first 8192")
    ap.add_argument("--profile-step", action="store_true",
                    help="warm up, run ONE step inside NVTX range 'timed_step', exit (for ncu)")
    return ap.parse_args()


def metric_name(L):
    return f"HE attention decode ms/token at L={L} (12 heads, d_head=64, n=8192)"


def _ring_desc():
    from paper_2602_08798_b200.backend import default_limbs, default_qbits

    L, qb = default_limbs(16384), default_qbits(16384)
    return (f"RNS-BFV N=16384, Q={L}x{qb}b primes, P {qb if qb <= 49 else qb + 1}b, dnum={L}, "
            f"{'FP64' if qb <= 49 else 'integer'}-pipe NTT")


def workload(args):
    """The config dict, identical in both arms (the GPU ring is reported beside it)."""
    return {"workload": f"decode_attention_{args.heads}h_L{args.L}", "heads": args.heads, "d_head": D2,
            "n_slots": N_SLOTS, "plain_modulus": P, "cached_len": args.L, "steps_appended": 1,
            "l2": "working set >1.5 GB per step (> 126 MB L2)", "parallelism": f"replicas{args.gpus}"}


# ----------------------------------------------------------------------------
# inputs (shared by all arms)
# ----------------------------------------------------------------------------
def fp_tokens(rng, rows, d):
    return np.mod(np.round(rng.uniform(-1.0, 1.0, (rows, d)) * (1 << F)).astype(np.int64), P)


def build_state(api, new_ctx, L, heads, seed=0):
    params = api.BackendParams()
    root = new_ctx(params, seed)
    fp = api.FixedPointParams(F, P)
    rng = np.random.default_rng(seed)
    ctxs = [root.fork() for _ in range(heads)]
    caches = []
    for c in ctxs:
        K = api.encode(fp_tokens(rng, L, D2), api.EncodingKind.OUTER, c)
        V = api.encode(fp_tokens(rng, L, D2), api.EncodingKind.OUTER, c)
        caches.append(api.init_cache(K, V, c))
    chans = [api.MpcChannel(P, seed=1000 + h) for h in range(heads)]
    return root, fp, ctxs, caches, chans, rng


def step_tokens(rng, heads):
    """Host plaintext q, k, v (slot vectors) of one step, per head."""
    return [np.concatenate([fp_tokens(rng, 1, D2)[0], np.zeros(N_SLOTS - D2, np.int64)]) for _ in range(3 * heads)]


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def max_over_ranks(x: float, world: int) -> float:
    """Max of a per-rank timing over all ranks (device tensors under NCCL,
    CPU tensors under gloo); the value every rank reports."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def prefill_state(api, new_ctx, args, seed=0):
    params = api.BackendParams()
    root = new_ctx(params, seed)
    fp = api.FixedPointParams(F, P)
    rng = np.random.default_rng(seed)
    ctxs = [root.fork() for _ in range(args.heads)]
    host = [[fp_tokens(rng, args.L, D2) for _ in range(3)] for _ in ctxs]
    return root, fp, ctxs, host


def prefill_config(args):
    return {"workload": f"prefill_attention_{args.heads}h_L{args.L}", "heads": args.heads, "d_head": D2,
            "n_slots": N_SLOTS, "plain_modulus": P, "prompt_len": args.L,
            "l2": "working set > 126 MB L2 (1.5k+ ciphertexts of 768 KiB per wave)",
            "parallelism": f"replicas{args.gpus}"}


def run_prefill(args):
    """Config 2: encrypted prefill Q.K^T and P.V for `heads` heads at prompt length L
    (arcc.prefill_attention_heads: all heads swept together)."""
    # the 12 heads' sweeps keep ~30k ciphertexts live plus the weight rows' resident
    # extensions (arcc.EXT_A_SWEEP)
    os.environ.setdefault("CGB_ARENA_GIB", "48")
    import torch

    import paper_2602_08798_b200 as api
    from paper_2602_08798_b200 import _native
    from paper_2602_08798_b200.backend import GpuContext

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    _native.build()
    root, fp, ctxs, host = prefill_state(api, GpuContext, args)
    ring = root.ring
    stream = torch.cuda.current_stream()
    ring.set_stream(stream.cuda_stream)
    chan_seed = [0]

    def chans():
        chan_seed[0] += 1
        return [api.MpcChannel(P, seed=2000 + 100 * chan_seed[0] + h) for h in range(args.heads)]

    def encrypt_all():
        return [[api.encode(x, api.EncodingKind.OUTER, c) for x in hq] for hq, c in zip(host, ctxs)]

    def run(mats):
        return api.prefill_attention_heads([m[0] for m in mats], [m[1] for m in mats], [m[2] for m in mats], fp,
                                           ctxs, chans())

    mats = encrypt_all()
    clk = ClockSampler(local).__enter__()  # started before the warm-up (its start-up stalls)
    run(mats)  # warm-up (key generation)
    gc.collect()
    gc.freeze()
    torch.cuda.synchronize()
    l0 = ring.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if True:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            run(mats)
        ev1.record(stream)
        torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = ring.launches() - l0
    # e2e: host plaintext Q, K, V -> client encryption -> prefill -> client decryption of the outputs
    h0, d0 = ring.h2d_bytes, ring.d2h_bytes
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        outs = run(encrypt_all())
        [api.decode(o, c) for o, c in zip(outs, ctxs)]
    ev1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = ev0.elapsed_time(ev1) / args.steps
    h2d, d2h = (ring.h2d_bytes - h0) / args.steps, (ring.d2h_bytes - d0) / args.steps
    roof, table, _ = unit_roofline(ring, lambda: run(mats), stream, _peaks(), ring.modmul_peak())
    line = {"metric": f"HE prefill attention ms (Q.K^T and P.V, {args.heads} heads, L={args.L})", "value": ms,
            "unit": "ms", "n_gpus": 1, "steps": args.steps, "warmup": 1, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded uniform [-1,1], f=8)", "config": prefill_config(args), "ring": _ring_desc(),
            "e2e": {"value": ms_e2e, "unit": "ms", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches), "roofline": roof, "units": table, "clocks": clk.summary()}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = prefill_cpu_baseline(args)
    print(json.dumps(line), flush=True)


def prefill_cpu_baseline(args):
    """ONE head of the same prefill on the reference's CPU path (per-op
    restatement oracle/reference_path.prefill_attention over the slot emulation),
    scaled to all heads (heads are independent and identical in op count)."""
    from oracle import reference_path as ref
    from oracle.slots import SlotContext
    import paper_2602_08798_b200 as api

    root, fp, ctxs, host = prefill_state(api, SlotContext, args)
    mats = [api.encode(x, api.EncodingKind.OUTER, ctxs[0]) for x in host[0]]
    t0 = time.perf_counter()
    ref.prefill_attention(*mats, fp, ctxs[0], api.MpcChannel(P, seed=2000))
    dt = time.perf_counter() - t0
    return {"value": dt * 1e3 * args.heads, "unit": "ms", "cores": 1, "kind": "port",
            "sample": f"1 of {args.heads} heads at L={args.L} timed ({dt:.1f} s), x{args.heads}; sequential per-op "
                      "slot emulation (oracle/reference_path.prefill_attention + oracle/slots.py)",
            "host": _cpu_model()}


GPT2_VOCAB = 50257


def layer_model(args):
    from paper_2602_08798_b200 import model as M

    cfg = M.ModelConfig(layers=1, d1=HEADS * D2, heads=HEADS, ffn_dim=4 * HEADS * D2, vocab=GPT2_VOCAB,
                        max_seq=args.L + args.steps + args.warmup + 2, f=F,
                        unembed_vocab=None if getattr(args, "full_vocab", False) else N_SLOTS)
    return M, M.gpt2_layer_model(cfg, seed=0)


def run_layer(args):
    """Config 3: one GPT-2-small decoder layer (d_model 768, 12 heads, d_ff 3072,
    N(0, 0.02) weights), a prompt of L token ids uniform over 50257, then
    `steps` greedy tokens, every cache part force-refreshed before each step.
    The unembedding covers the first 8192 vocabulary entries (n_slots)."""
    # the FFN prefill keeps ~20k ciphertexts live; every decode-step weight diagonal stays
    # resident (a full-vocabulary unembedding: 7 x 8192 diagonals, 57k products per token)
    # plaintext arena: every decode-side weight diagonal (~33k: 36 head projections x 768,
    # wo, w1, w2, the unembedding) stays resident next to the forced refresh's 3.1k mask
    # plaintexts per token; at 12 GiB the masks evicted diagonals (a 1.4 s re-encode token)
    # (~8k rotation keys of 6 MiB stay resident too: arenas + keys + workspace < 180 GB)
    os.environ.setdefault("CGB_ARENA_GIB", "48")
    os.environ.setdefault("CGB_PT_ARENA_GIB", "34" if args.full_vocab else "24")
    import torch

    from paper_2602_08798_b200 import _native
    from paper_2602_08798_b200.backend import BackendParams, GpuContext

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    _native.build()
    M, mdl = layer_model(args)
    ctx = GpuContext(BackendParams(), 0)
    ring = ctx.ring
    stream = torch.cuda.current_stream()
    ring.set_stream(stream.cuda_stream)
    prompt = np.random.default_rng(0).integers(0, GPT2_VOCAB, args.L).tolist()
    chans = M.channels(0, 1, HEADS, P)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 2)]
    torch.cuda.synchronize()
    l0 = ring.launches()
    t0 = time.perf_counter()
    ev[0].record(stream)
    state = M.prefill(mdl, prompt, ctx, chans)
    ev[1].record(stream)
    torch.cuda.synchronize()
    t_pre = time.perf_counter() - t0
    pre_ms = ev[0].elapsed_time(ev[1])
    # warm-up decode token(s): the first builds the decode-side weight diagonals (a
    # one-time model setup) and every rotation key of the step; timed separately
    first_ms = []
    toks = []
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))).__enter__()  # before the warm-up token
    for _ in range(max(1, args.warmup)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tok, state = M.decode_step(mdl, state, ctx, chans, force_refresh=True)
        toks.append(tok)
        e1.record(stream)
        torch.cuda.synchronize()
        first_ms.append(e0.elapsed_time(e1))
    l1 = ring.launches()
    gc.collect()
    gc.freeze()
    h0, d0 = ring.h2d_bytes, ring.d2h_bytes
    torch.cuda.synchronize()
    ev[1].record(stream)  # the timed tokens start here (after the warm-up tokens)
    if True:
        for i in range(args.steps):
            tok, state = M.decode_step(mdl, state, ctx, chans, force_refresh=True)
            toks.append(tok)
            ev[i + 2].record(stream)
        torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    t_all = time.perf_counter() - t0
    h2d, d2h = (ring.h2d_bytes - h0) / args.steps, (ring.d2h_bytes - d0) / args.steps
    step_ms = [ev[i + 1].elapsed_time(ev[i + 2]) for i in range(args.steps)]
    # one more step outside the timed ones with CUDA events around every launch
    ring.timing(True)
    M.decode_step(mdl, state, ctx, chans, force_refresh=True)
    torch.cuda.synchronize()
    rep = ring.timing_report()
    ring.timing(False)
    kern = {k: {"launches": v[0], "ms": round(v[1], 3)} for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1])}
    roof, table, _ = unit_roofline(ring, lambda: M.decode_step(mdl, state, ctx, chans, force_refresh=True), stream,
                                   _peaks(), ring.modmul_peak())
    line = {"metric": f"HE decoder-layer decode ms/token (GPT-2 small layer, prompt {args.L}, "
                      f"{args.steps} tokens, refresh each step)",
            # value: mean decode ms/token over the timed tokens, after `warmup` untimed tokens
            # (the first builds the decode-side weight diagonals once: first_token_ms)
            "value": float(np.mean(step_ms)), "unit": "ms/token", "higher_is_better": False, "n_gpus": 1,
            "warmup_tokens": len(first_ms), "first_token_ms": first_ms,
            "e2e": {"value": float(np.mean(step_ms)), "unit": "ms/token", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "note": "decode_step is end to end: host token id in, client-decrypted logits out"},
            "roofline": roof, "units": table, "clocks": clk.summary(),
            "steps": args.steps, "dtype": "u64", "data": "synthetic (token ids uniform over 50257, N(0,0.02) weights)",
            "config": {"workload": f"gpt2_layer_prompt{args.L}_gen{args.steps}", "d_model": HEADS * D2,
                       "heads": HEADS, "d_ff": 4 * HEADS * D2, "vocab": GPT2_VOCAB, "unembed_vocab": GPT2_VOCAB if args.full_vocab else N_SLOTS,
                       "n_slots": N_SLOTS, "plain_modulus": P, "ring": _ring_desc()},
            "prefill_ms": pre_ms, "decode_ms_per_token": step_ms,
            "wall_s": {"prefill": t_pre, "total": t_all},
            "gpu_launches": {"prefill": int(l1 - l0), "decode_per_token": int((ring.launches() - l1) / args.steps)},
            "tokens": toks, "counters": ctx.counter.as_dict(),
            "kernels_one_step": kern}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = layer_cpu_baseline(args)
    print(json.dumps(line), flush=True)


def layer_cpu_baseline(args):
    """One decode step of the same layer on the reference's CPU path (this
    package's host code over the slot emulation, oracle/slots.py), with the
    caches built directly by encode (config 4's shortcut) instead of a prefill."""
    from oracle.slots import SlotContext
    import paper_2602_08798_b200 as api
    from paper_2602_08798_b200.backend import BackendParams

    M, mdl = layer_model(args)
    ctx = SlotContext(BackendParams(), 0)
    rng = np.random.default_rng(0)
    caches = [[api.init_cache(*(api.encode(fp_tokens(rng, args.L, D2), api.EncodingKind.OUTER, ctx)
                                for _ in range(2)), ctx) for _ in range(HEADS)]]
    state = M.GenerationState(position=args.L, caches=caches, next_logits=np.zeros(8, np.int64))
    chans = M.channels(0, 1, HEADS, P)
    t0 = time.perf_counter()
    M.decode_step(mdl, state, ctx, chans, force_refresh=True)
    dt = time.perf_counter() - t0
    return {"value": dt * 1e3, "unit": "ms/token", "cores": 1, "kind": "port",
            "sample": f"one decode step of the layer at cached length {args.L} (caches by encode), slot emulation",
            "host": _cpu_model()}


def unit_roofline(ring, step, stream, hbm_peak: float, peak_mm: float):
    """Run `step` once with every multi-launch operation timed as one unit
    (cgb_timing_enable 2, PDL on inside) and return (roofline dict of the batched
    key switch per SURVEY 8(d), units table, timed step ms)."""
    import torch

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ring.timing(2)
    ev0.record(stream)
    step()
    ev1.record(stream)
    units = ring.timing_report()
    ring.timing(0)
    unit_step_ms = ev0.elapsed_time(ev1)
    ks = [units[k] for k in ("keyswitch", "keyswitch_hoisted") if k in units]
    nl, kms = sum(v[0] for v in ks), sum(v[1] for v in ks)
    kbytes, kmm = sum(v[2] for v in ks), sum(v[3] for v in ks)
    achieved = kbytes / (kms * 1e-3) / 1e9 if kms else 0.0
    roof = {"bound": "hbm", "kernel": "keyswitch (batched hybrid key switch as one unit: 5 fused launches, "
                                      "or the hoisted variant)",
            "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
            "traffic": _traffic_ks(kbytes / nl if nl else 0.0, ring), "launches_per_step": nl,
            "bytes_per_launch": kbytes / nl if nl else None,
            "bytes_def": "per batch: (input ct + output ct) x items + 2 dnum (L+1) N x 8 B per distinct key",
            "share_of_step": kms / unit_step_ms if unit_step_ms else None,
            "timing": "CUDA events around each whole batched key switch, PDL on inside (cgb_timing_enable 2)",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)",
            "pipe": {"name": "fp64" if ring.fp_ntt else "int64", "unit": "modmul/s",
                     "achieved": kmm / (kms * 1e-3) if kmm else None, "peak": peak_mm,
                     "frac": kmm / (kms * 1e-3) / peak_mm if kmm else None,
                     "peak_source": "cgb_modmul_peak: measured chains of the same modular product"}}
    table = {k: {"calls": v[0], "ms": round(v[1], 3), "GBps": round(v[2] / (v[1] * 1e-3) / 1e9, 1) if v[1] else None,
                 "Gmodmul_s": round(v[3] / (v[1] * 1e-3) / 1e9, 1) if v[1] and v[3] else None}
             for k, v in sorted(units.items(), key=lambda kv: -kv[1][1]) if not k.startswith("(")}
    return roof, table, unit_step_ms


def _peaks():
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    return peaks.get("hbm_gbs", 6650.0)


def _traffic_ks(alg_bytes_per_launch: float, ring):
    """DRAM bytes per batched key switch from the committed ncu --set full capture of
    its five kernels (profiles/r02/ncu_keyswitch.json: DRAM bytes per key-switched
    item), scaled to this bench's average batch; None without a capture."""
    f = ROOT / "profiles" / "r02" / "ncu_keyswitch.json"
    if not f.exists():
        return None
    cap = json.loads(f.read_text())
    per_item, alg_item = cap.get("dram_bytes_per_item"), cap.get("algorithmic_bytes_per_item")
    if not per_item or not alg_item:
        return None
    return {"bytes_per_launch": alg_bytes_per_launch * per_item / alg_item,
            "dram_over_algorithmic": per_item / alg_item, "source": "profiles/r02/ncu_keyswitch.json"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2602_08798_b200 as api
    from paper_2602_08798_b200 import _native

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    _native.build()
    from paper_2602_08798_b200.backend import GpuContext

    root, fp, ctxs, caches, chans, rng = build_state(api, GpuContext, args.L, args.heads, seed=rank)
    ring = root.ring
    stream = torch.cuda.current_stream()
    ring.set_stream(stream.cuda_stream)
    C = GpuContext
    W = args.warmup + args.steps
    host_tokens = [step_tokens(rng, args.heads) for _ in range(W)]
    # device-resident inputs for the `value` leg
    dev_tokens = []
    for toks in host_tokens:
        w = C.w_encrypt([c for c in ctxs for _ in range(3)], np.stack(toks)).handles()
        dev_tokens.append(w)

    def one_step(tok_handles):
        qs, ks, vs = tok_handles[0::3], tok_handles[1::3], tok_handles[2::3]
        cs = api.maybe_refresh_heads(caches, ctxs, chans)
        cs = api.append_token_heads(cs, ks, vs, ctxs)
        return api.attention_step_heads(qs, cs, fp, ctxs, chans)

    def one_step_e2e(toks):
        wave = C.w_encrypt([c for c in ctxs for _ in range(3)], np.stack(toks))
        outs = one_step(wave.handles())
        return C.w_decrypt(C.wave_of(outs, ctxs))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        one_step(dev_tokens[i])
        if i == 0:
            # the setup's long-lived objects (caches, keys, tables) out of the cyclic
            # GC's generations: a full collection over them inside the timed loop is a
            # host stall; the remaining warm-up steps run after the freeze
            gc.collect()
            gc.freeze()
    if args.profile_step:
        barrier()
        torch.cuda.nvtx.range_push("timed_step")
        one_step(dev_tokens[args.warmup])
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        print(json.dumps({"profile_step": "done", "launches": ring.launches()}))
        return
    # the clock sampler (an nvidia-smi child) starts BEFORE the last warm-up step: its
    # start-up (NVML init on this GPU) once stalled the first timed step by 150-250 ms
    clk = ClockSampler(local).__enter__()
    one_step_e2e(host_tokens[0])
    one_step(dev_tokens[args.warmup - 1])
    barrier()
    launches0 = ring.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if True:
        barrier()
        ev0.record(stream)
        marks = []
        for i in range(args.steps):
            one_step(dev_tokens[args.warmup + i])
            marks.append((torch.cuda.Event(enable_timing=True), time.perf_counter()))
            marks[-1][0].record(stream)
        ev1.record(stream)
        barrier()
    clk.__exit__(None, None, None)
    ms = ev0.elapsed_time(ev1)
    dev = [round((marks[0][0] if i == 0 else marks[i - 1][0]).elapsed_time(marks[i][0]), 2) if i else
           round(ev0.elapsed_time(marks[0][0]), 2) for i in range(len(marks))]
    wall = [round(1e3 * (marks[i][1] - (marks[i - 1][1] if i else marks[0][1])), 2) for i in range(len(marks))]
    if os.environ.get("CGB_BENCH_STEPTIMES") or max(dev) > 1.1 * statistics.median(dev):
        print("per-step device ms:", dev, file=sys.stderr)
        print("per-step host ms:", wall, file=sys.stderr)
    launches = ring.launches() - launches0
    # e2e leg: host plaintext in, host plaintext out
    h0, d0 = ring.h2d_bytes, ring.d2h_bytes
    barrier()
    ev0.record(stream)
    for i in range(args.steps):
        one_step_e2e(host_tokens[args.warmup + i])
    ev1.record(stream)
    barrier()
    ms_e2e = ev0.elapsed_time(ev1)
    h2d = (ring.h2d_bytes - h0) / args.steps
    d2h = (ring.d2h_bytes - d0) / args.steps
    # live timing passes, one step each: (1) CUDA events around every launch (PDL off:
    # the per-kernel table); (2) events around every multi-launch operation -- a whole
    # batched key switch, a whole mult_cipher -- with PDL on inside it (the 8(d) units
    # the roofline is computed on)
    ring.timing(1)
    one_step(dev_tokens[args.warmup])
    rep = ring.timing_report()
    ring.timing(2)
    ev0.record(stream)
    one_step(dev_tokens[args.warmup])
    ev1.record(stream)
    units = ring.timing_report()
    ring.timing(0)
    unit_step_ms = ev0.elapsed_time(ev1)
    idle_ms = rep.pop("(idle)", (0, 0.0, 0.0))[1]
    gaps = {k: round(v[1], 3) for k, v in rep.items() if k.startswith("(gap")}
    for k in gaps:
        rep.pop(k)
    trans = {k[7:-1]: [v[0], round(v[1], 3)] for k, v in rep.items() if k.startswith("(trans:")}
    for k in list(rep):
        if k.startswith("(trans:"):
            rep.pop(k)
    peak_mm = ring.modmul_peak()

    ms, ms_e2e = max_over_ranks(ms, world), max_over_ranks(ms_e2e, world)
    if rank != 0:
        dist.destroy_process_group()
        return
    ms_step = ms / args.steps
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    step_kernel_ms = sum(v[1] for v in rep.values())
    # the dominant unit: the batched key switch (five fused launches, or the hoisted
    # variant), bytes = inputs + outputs once + each distinct key once
    ks = [units[k] for k in ("keyswitch", "keyswitch_hoisted") if k in units]
    nl, kms = sum(v[0] for v in ks), sum(v[1] for v in ks)
    kbytes, kmm = sum(v[2] for v in ks), sum(v[3] for v in ks)
    achieved = kbytes / (kms * 1e-3) / 1e9
    mc = [units[k] for k in ("mult_cipher", "mult_cipher_ext") if k in units]
    # arithmetic pipe (FP64 exact products for rings of < 2^49 primes, else 64-bit Shoup):
    # algorithmic modular products (butterflies + key / constant products) per second
    arith = [v for v in rep.values() if v[3] > 0]
    ar_ms, ar_mm = sum(v[1] for v in arith), sum(v[3] for v in arith)
    line = {
        # value: per-token latency of the job; N > 1 runs N independent replicas,
        # each producing one token per step, timed as the max over ranks
        "metric": metric_name(args.L), "value": ms_step, "unit": "ms/token", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded uniform [-1,1], f=8)",
        "config": workload(args), "ring": _ring_desc(),
        "e2e": {"value": ms_e2e / args.steps, "unit": "ms/token", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "keyswitch (batched hybrid key switch as one unit: 5 fused "
                                               "launches, or the hoisted variant)",
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                     "traffic": _traffic_ks(kbytes / nl if nl else 0.0, ring), "launches_per_step": nl,
                     "bytes_per_launch": kbytes / nl if nl else None,
                     "bytes_def": "per batch: (input ct + output ct) x items + 2 dnum (L+1) N x 8 B per distinct key",
                     "share_of_step": kms / unit_step_ms if unit_step_ms else None,
                     "timing": "CUDA events around each whole batched key switch, PDL on inside (cgb_timing_enable 2)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)",
                     "pipe": {"name": "fp64" if ring.fp_ntt else "int64", "unit": "modmul/s",
                              "achieved": kmm / (kms * 1e-3) if kmm else None, "peak": peak_mm,
                              "frac": kmm / (kms * 1e-3) / peak_mm if kmm else None,
                              "peak_source": "cgb_modmul_peak: measured chains of the same modular product"}},
        "units": {k: {"calls": v[0], "ms": round(v[1], 3), "GBps": round(v[2] / (v[1] * 1e-3) / 1e9, 1) if v[1] else None,
                      "Gmodmul_s": round(v[3] / (v[1] * 1e-3) / 1e9, 1) if v[1] and v[3] else None}
                  for k, v in sorted(units.items(), key=lambda kv: -kv[1][1]) if not k.startswith("(")},
        "mult_cipher_unit": {"ms": sum(v[1] for v in mc), "GBps": sum(v[2] for v in mc) / (sum(v[1] for v in mc) * 1e-3) / 1e9
                             if mc else None},
        "arith_pipe": {"kernels": "every launch with modular-product work (NTT passes, fused key switch)",
                       "pipe": "fp64" if ring.fp_ntt else "int64",
                       "modmuls_per_s": ar_mm / (ar_ms * 1e-3) if ar_ms else None,
                       "peak_modmuls_per_s": peak_mm,
                       "frac": ar_mm / (ar_ms * 1e-3) / peak_mm if ar_ms else None,
                       "share_of_step": ar_ms / step_kernel_ms if step_kernel_ms else None},
        "kernels": {k: {"launches": v[0], "ms": round(v[1], 4),
                        "GBps": round(v[2] / (v[1] * 1e-3) / 1e9, 1) if v[1] else None,
                        "Gmodmul_s": round(v[3] / (v[1] * 1e-3) / 1e9, 1) if v[1] and v[3] else None}
                    for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1])},
        "clocks": clk.summary(),
        "step_ms": dev,
        "gpu_idle_ms_per_step": round(idle_ms, 2),
        "gpu_idle_top_gaps_ms": gaps,
        "gpu_idle_by_transition_ms": trans,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, samples=3)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------
# reference arm: the reference's CPU path (sequential per-op, slot emulation)
# ----------------------------------------------------------------------------
def reference_step_fn(args):
    from oracle import reference_path as ref
    from oracle.slots import SlotContext
    import paper_2602_08798_b200 as api

    root, fp, ctxs, caches, chans, rng = build_state(api, SlotContext, args.L, args.heads, seed=0)

    def step():
        toks = step_tokens(rng, args.heads)
        outs = []
        for h in range(args.heads):
            c = ctxs[h]
            q, k, v = (c.encrypt(toks[3 * h + j]) for j in range(3))
            cache = ref.maybe_refresh(caches[h], c, chans[h])
            cache = ref.append_token(cache, k, v, c)
            outs.append(c.decrypt(ref.attention_step(q, cache, fp, c, chans[h])))
        return outs

    return step


def cpu_baseline(args, samples=1):
    step = reference_step_fn(args)
    step()  # warm
    ts = []
    for _ in range(samples):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    return {"value": min(ts) * 1e3, "unit": "ms/token", "cores": 1, "kind": "port",
            "sample": f"{args.heads}-head decode step at L={args.L}, sequential per-op slot emulation "
                      f"(oracle/reference_path.py + oracle/slots.py), best of {samples}",
            "host": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" x{os.cpu_count()}"
    except OSError:
        pass
    return None


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    step = reference_step_fn(args)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    line = {"impl": "reference", "metric": metric_name(args.L), "value": ms, "unit": "ms/token", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64 (Z_p slot emulation)", "data": "synthetic",
            "config": workload(args),
            "cpu_baseline": {"value": ms, "unit": "ms/token", "cores": 1, "kind": "port",
                             "sample": f"{args.steps} decode steps x {args.heads} heads at L={args.L}",
                             "host": _cpu_model()},
            "e2e": {"value": ms, "unit": "ms/token", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.workload == "prefill":
        run_prefill(a)
    elif a.workload == "layer":
        run_layer(a)
    else:
        run_ours(a)
