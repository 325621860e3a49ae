"""Recompute the bench line's key-switch roofline from DESIGN.md §4.1's units and
the committed ncu launch list (the verdict's check: bench `roofline.frac` vs a
recompute from profiles/ within 5 %).

    python scripts/roofline_recompute.py [bench.json] [launches.csv]

Key-switch unit time from ncu: every five-kernel group ks_digit_rows ->
col_fused -> ks_row<..,1> -> col_fused -> ks_row<..,2> (or k_ks_row2) that is NOT a
relinearisation (a relinearisation's digit-rows pass directly follows the
forward NTT row pass of mult_cipher's scale-and-round output), summed.
Bytes: the bench line's own 8(d) bytes per step (launches_per_step x
bytes_per_launch), i.e. the units DESIGN.md §4.1 defines.  ncu durations are
cold-cache and serialised, so the two times agree only to a few percent.
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
bench = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r02" / "bench_full.json"
launches = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "profiles" / "r02" / "launches_decode.csv"

line = json.loads(bench.read_text().strip().splitlines()[-1])
roof = line["roofline"]
rows = [r for r in csv.reader(open(launches)) if len(r) > 10 and r[0].isdigit()]
names = [r[6].split("(")[0].replace("void ", "").replace("cgb::", "") for r in rows]
ns = [float(r[-1]) for r in rows]
seq = (("k_ntt2_fpr<7, 7, 0, 1",), ("k_col_fused",), ("k_ks_row<7, 7, 3, 1", "k_ks_row2<7, 7, 3, 0"), ("k_col_fused",),
       ("k_ks_row<7, 7, 3, 2", "k_ks_row2<7, 7, 3, 1"))
ks_ns, relin_ns, groups, relin = 0.0, 0.0, 0, 0
i = 0
while i + 5 <= len(names):
    if all(names[i + k].startswith(seq[k]) for k in range(5)):  # str.startswith takes a tuple of alternatives
        t = sum(ns[i:i + 5])
        if i > 0 and names[i - 1].startswith("k_ntt2_fpr<7, 7, 1, 1"):
            relin_ns += t
            relin += 1
        else:
            ks_ns += t
            groups += 1
        i += 5
    else:
        i += 1
step_bytes = roof["launches_per_step"] * roof["bytes_per_launch"]
achieved = step_bytes / (ks_ns * 1e-9) / 1e9
frac = achieved / roof["peak"]
out = {"bench_frac": roof["frac"], "recomputed_frac": frac, "rel_diff": frac / roof["frac"] - 1.0,
       "ncu_keyswitch_ms": ks_ns / 1e6, "ncu_groups": groups, "bench_launches_per_step": roof["launches_per_step"],
       "relinearisation_groups_excluded": relin, "relinearisation_ms": relin_ns / 1e6,
       "bytes_per_step": step_bytes, "peak_GBps": roof["peak"]}
print(json.dumps(out, indent=1))
