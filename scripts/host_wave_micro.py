"""Host cost of one small key-switch wave (12 items) vs its GPU time."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_08798_b200.backend import BackendParams, GpuContext  # noqa: E402

ctx = GpuContext(BackendParams(), 0)
C = GpuContext
for items in (12, 768):
    w = C.w_encrypt([ctx] * items, np.zeros((items, 8192), np.int64))
    for step in (1, 2):
        C.w_rotate(w, step, add_input=True)
    torch.cuda.synchronize()
    reps = 50 if items == 12 else 5
    t0 = time.perf_counter()
    for i in range(reps):
        C.w_rotate(w, 1 + (i % 2), add_input=True)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{items} items: host enqueue {1e6 * (t1 - t0) / reps:.1f} us/wave, "
          f"enqueue+drain {1e6 * (t2 - t0) / reps:.1f} us/wave", flush=True)
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for i in range(reps):
        C.w_rotate(w, 1 + (i % 2), add_input=True)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(8)
