import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2602_08798_b200 import _native
from paper_2602_08798_b200.ring import Ring
_native.build()
for (logn, t, L, n, row) in [(3, 17, 8, 4, True), (3, 17, 2, 4, True), (4, 97, 8, 8, True), (4, 1048609, 8, 16, False)]:
    try:
        r = Ring(logn, t, L, n, row, np.arange(8, dtype=np.uint32), arena_cts=16, arena_pts=8)
        ids = r.alloc(2)
        r.encrypt(np.arange(n), np.arange(8, dtype=np.uint32), 0, ids[:1])
        print(logn, t, L, n, row, "ok", r.decrypt(ids[:1])[0][:4])
    except Exception as e:
        print(logn, t, L, n, row, "FAIL", e)
