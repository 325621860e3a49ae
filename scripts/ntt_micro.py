"""NTT microbench: per-launch time of the batched forward / inverse NTT on
uniform (zero) data at the decode ring (logN 14, 3 x 49-bit limbs)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_08798_b200.ring import Ring
from bench_kernels import plain_modulus_for

logn = int(os.environ.get("LOGN", 14)); N = 1 << logn
L = int(os.environ.get("CGB_LIMBS", 3)); qb = int(os.environ.get("CGB_QBITS", 49))
ring = Ring(logn, plain_modulus_for(N), L, N // 2, True, np.arange(8, dtype=np.uint32), q_bits=qb)
B = int(os.environ.get("BATCH", 36)); iters = int(os.environ.get("ITERS", 50))
for fwd in (True, False):
    ms = ring.bench_ntt(B, fwd, iters)
    polys = B * 2 * L
    print(json.dumps({"variant": os.environ.get("VARIANT", ""), "dir": "fwd" if fwd else "inv", "polys": polys,
                      "us": ms * 1e3, "ns_per_poly": ms * 1e6 / polys,
                      "GBps": polys * N * 8 * 4 / (ms * 1e-3) / 1e9}), flush=True)
