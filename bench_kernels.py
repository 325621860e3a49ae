"""Kernel microbenchmark: batched NTT/INTT, pointwise
RNS modmul and hybrid key switching at N = 2^13 .. 2^16 with 2-8 primes of
~50 bits, batch 64 ciphertexts, residues uniform.  One JSON line per case.

Rooflines: NTT against the measured peak of the same modular product on the
pipe the ring uses (cgb_modmul_peak: the FP64 error-free product for primes
< 2^49, else the 64-bit integer Shoup product) and against HBM for its
algorithmic bytes (read + write each limb-poly once); pointwise ops, key
switching and mult_cipher against the measured HBM copy bandwidth
(MEASURED_PEAKS.json), the key switch also against the modular-product pipe.
Every line carries the nvidia-smi clocks sampled during the sweep.
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def plain_modulus_for(N):
    from paper_2602_08798_b200.backend import is_prime

    c = (1 << 29) + 1
    c += (-(c - 1)) % (2 * N)
    while not is_prime(c):
        c += 2 * N
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logn", default="13,14,15,16")
    ap.add_argument("--limbs", default="2,3,4,5,6,8")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--qbits", type=int, default=49)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    import torch

    from paper_2602_08798_b200 import _native
    from paper_2602_08798_b200.ring import Ring

    _native.build()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    stream = torch.cuda.current_stream()
    peak_mm = None
    from bench import ClockSampler

    clk = ClockSampler(0).__enter__()  # nvidia-smi clocks + throttle reasons over the whole sweep

    def emit(d):
        d["clocks"] = clk.summary()
        print(json.dumps(d), flush=True)

    for logn in [int(x) for x in a.logn.split(",")]:
        N = 1 << logn
        for L in [int(x) for x in a.limbs.split(",")]:
            ring = Ring(logn, plain_modulus_for(N), L, N // 2, True, np.arange(8, dtype=np.uint32),
                        arena_cts=3 * a.batch + 4, arena_pts=a.batch + 4, q_bits=a.qbits)
            ring.set_stream(stream.cuda_stream)
            if peak_mm is None:
                peak_mm = ring.modmul_peak()
            B = a.batch
            polys = B * 2 * L
            for fwd in (True, False):
                ms = ring.bench_ntt(B, fwd, a.iters)
                bfly = polys * (N // 2) * logn
                by = polys * N * 8 * 2
                emit({"kernel": "ntt_fwd" if fwd else "ntt_inv", "logN": logn, "limbs": L, "q_bits": a.qbits,
                      "batch_cts": B, "ms": ms, "butterflies_per_s": bfly / (ms * 1e-3),
                      "modmul_pipe_frac": bfly / (ms * 1e-3) / peak_mm, "GBps": by / (ms * 1e-3) / 1e9,
                      "hbm_frac": by / (ms * 1e-3) / 1e9 / hbm,
                      "pipe": "fp64" if ring.fp_ntt else "int64 (Shoup)"})
            # pointwise mult_plain and key switching (one shared Galois key) on uniform ciphertexts
            rng = np.random.default_rng(logn * 10 + L)
            ids = ring.alloc(3 * B)
            src, dst, tmp = ids[:B], ids[B:2 * B], ids[2 * B:]
            words = np.stack([np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in ring.moduli[:L]])
                              for _ in range(2)])
            ring.load(src, np.broadcast_to(words, (B, 2, L, N)))
            ring.load(tmp, np.broadcast_to(words, (B, 2, L, N)))
            pts = ring.alloc_pt(B)
            ring.encode_pt(rng.integers(0, ring.t, (B, N // 2)), 0, pts)
            ring.prepare_galois([ring.galois_elt(1)])
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

            def timed(fn):
                fn()
                torch.cuda.synchronize()
                ev[0].record(stream)
                for _ in range(a.iters):
                    fn()
                ev[1].record(stream)
                torch.cuda.synchronize()
                return ev[0].elapsed_time(ev[1]) / a.iters

            ct_b = 2 * L * N * 8
            ms = timed(lambda: ring.mult_plain(src, pts, dst))
            by = B * (2 * ct_b + L * N * 8)
            emit({"kernel": "mult_plain", "logN": logn, "limbs": L, "batch_cts": B, "ms": ms,
                  "GBps": by / (ms * 1e-3) / 1e9, "hbm_frac": by / (ms * 1e-3) / 1e9 / hbm})
            ms = timed(lambda: ring.rotate(src, [1], dst))
            ring.timing(2)  # modular products of one batched key switch (the unit's report)
            ring.rotate(src, [1], dst)
            unit = ring.timing_report().get("keyswitch", (1, ms, 0.0, 0.0))
            ring.timing(0)
            evk = 2 * L * (L + 1) * N * 8
            by = evk + B * 2 * ct_b
            emit({"kernel": "keyswitch_rotate", "logN": logn, "limbs": L, "dnum": L, "batch_cts": B, "ms": ms,
                  "us_per_ct": ms * 1e3 / B, "GBps": by / (ms * 1e-3) / 1e9,
                  "hbm_frac": by / (ms * 1e-3) / 1e9 / hbm,
                  "modmul_pipe_frac": unit[3] / (unit[1] * 1e-3) / peak_mm if unit[3] else None,
                  "fused": L <= 8 and ring.fp_ntt, "limb_transforms_per_ct": 4 * L + 2 + (L - 1) * L})
            ms = timed(lambda: ring.mult_cipher(src, tmp, dst))
            by = B * 3 * ct_b + evk
            emit({"kernel": "mult_cipher", "logN": logn, "limbs": L, "batch_cts": B, "ms": ms,
                  "us_per_ct": ms * 1e3 / B, "GBps": by / (ms * 1e-3) / 1e9, "hbm_frac": by / (ms * 1e-3) / 1e9 / hbm})
            ring.free(ids)
            ring.free_pt(pts)
            ring.close()
    clk.__exit__()


if __name__ == "__main__":
    main()
