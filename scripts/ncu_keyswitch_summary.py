"""Summarise gpurun_out/prof_ks_raw.csv (ncu --set full of ONE batched key switch,
scripts/gpu_ks_profile.sh) into profiles/<round>/ncu_keyswitch.{json,md}: per-kernel
time, registers, DRAM bytes, FP64-pipe / LSU-data-pipe / issue utilisation, and the DRAM
bytes per key-switched ciphertext that bench.py reports as the roofline's `traffic`."""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
src = ROOT / "gpurun_out" / "prof_ks_raw.csv"
rows = list(csv.reader(src.open()))
h, units, data = rows[0], rows[1], rows[2:]
ix = {k: i for i, k in enumerate(h)}
KEEP = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
]
def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None
kern = []
for r in data:
    d = {"kernel": r[ix["Kernel Name"]].split("(")[0]}
    for k in KEEP:
        if k in ix:
            d[k] = num(r[ix[k]])
            if k.startswith("dram__bytes"):  # normalise to MB
                u = units[ix[k]]
                d[k] = d[k] * {"Gbyte": 1e3, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6}[u]
            if k == "gpu__time_duration.sum":
                d[k] = d[k] * {"us": 1.0, "ms": 1e3, "ns": 1e-3, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}[units[ix[k]]]
    kern.append(d)
# group the launches of one chunk: a chunk starts at the digit-rows kernel (k_ntt2_fpr inverse row pass)
chunks, cur = [], None
for d in kern:
    if "k_ntt2_fpr" in d["kernel"] or cur is None:
        cur = []
        chunks.append(cur)
    cur.append(d)
LOGN, L = 14, 3
ct_bytes = 2 * L * (1 << LOGN) * 8
key_bytes = 2 * L * (L + 1) * (1 << LOGN) * 8
out_chunks = []
for c in chunks:
    # items: the Q-limb row kernel's grid = items * L * 8 tiles
    last = c[-1]
    items = int(last["launch__grid_size"] // (L * 8))
    dr = sum(d["dram__bytes_read.sum"] for d in c)
    dw = sum(d["dram__bytes_write.sum"] for d in c)
    out_chunks.append({"items": items, "dram_read_MB": dr, "dram_write_MB": dw,
                       "us": sum(d["gpu__time_duration.sum"] for d in c),
                       "dram_bytes_per_item": (dr + dw) * 1e6 / items})
items = sum(c["items"] for c in out_chunks)
per_item = sum((c["dram_read_MB"] + c["dram_write_MB"]) for c in out_chunks) * 1e6 / items
alg = 2 * ct_bytes + key_bytes / items * len(out_chunks)
res = {"source": "ncu --set full --clock-control none of ONE batched key switch (scripts/gpu_ks_profile.sh: "
                 f"{items} items, rotate_add, logN 14, L 3, one Galois key; {len(out_chunks)} chunk(s))",
       "units": {"dram": "MB", "time": "us"}, "kernels": kern, "chunks": out_chunks,
       "dram_bytes_per_item": per_item, "algorithmic_bytes_per_item": 2 * ct_bytes + key_bytes / items * len(out_chunks),
       "dram_over_algorithmic": per_item / alg}
dst = ROOT / "profiles" / rnd
(dst / "ncu_keyswitch.json").write_text(json.dumps(res, indent=1))
c0 = chunks[0]
md = [f"# ncu --set full: one batched key switch ({rnd}, after the row-kernel rework)\n",
      f"`scripts/gpu_ks_profile.sh` -> `scripts/ncu_keyswitch_summary.py`; first chunk ({out_chunks[0]['items']} items), "
      "`--clock-control none`, cold-cache serialised.\n",
      "| kernel | us | regs | warps active % | issue active % | FP64 pipe % | LSU data pipe % | long-scoreboard / issue | DRAM % of peak | DRAM MB r / w |",
      "|---|---|---|---|---|---|---|---|---|---|"]
for d in c0:
    g = lambda k: d.get(k)
    md.append(f"| `{d['kernel']}` | {g('gpu__time_duration.sum'):.1f} | {g('launch__registers_per_thread'):.0f} | "
              f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | {g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{g('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{g('l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed'):.1f} | "
              f"{g('smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio'):.2f} | "
              f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
              f"{g('dram__bytes_read.sum'):.0f} / {g('dram__bytes_write.sum'):.0f} |")
md.append(f"\nPer key-switched ciphertext: **{per_item / 1e6:.2f} MB of DRAM traffic against {alg / 1e6:.3f} MB algorithmic** "
          f"({per_item / alg:.2f}x).\n")
(dst / "ncu_keyswitch.md").write_text("\n".join(md))
print("\n".join(md))
