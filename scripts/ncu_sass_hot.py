"""Summarise an ncu --page source --csv --print-source sass dump: shared-memory
excess wavefronts, global sector excess and warp-stall samples per instruction."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
print(rows[0][1])
print("-- shared excess wavefronts")
for r in sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))[:8]:
    if f(r, "L1 Wavefronts Shared Excessive") > 0:
        print(" ", r[1].strip()[:58].ljust(58), f(r, "L1 Wavefronts Shared"), f(r, "L1 Wavefronts Shared Ideal"))
print("-- global sector excess")
for r in sorted(data, key=lambda r: -f(r, "L2 Theoretical Sectors Global Excessive"))[:5]:
    if f(r, "L2 Theoretical Sectors Global Excessive") > 0:
        print(" ", r[1].strip()[:58].ljust(58), f(r, "L2 Theoretical Sectors Global"), f(r, "L2 Theoretical Sectors Global Ideal"))
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print("-- stall samples (total %d)" % tot)
seen = set()
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)")):
    if r[0] in seen: continue
    seen.add(r[0])
    if len(seen) > 12: break
    print(" ", r[1].strip()[:58].ljust(58), f(r, "Warp Stall Sampling (All Samples)"))
