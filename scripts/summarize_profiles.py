"""Turn ncu outputs in gpurun_out/ into committed summaries under profiles/<round>/.

  launches.csv  (ncu --metrics gpu__time_duration.sum --csv)  -> launch_share.md
  prof_*.ncu-rep (ncu --set full)                              -> ncu_<tag>.md
"""
import collections
import csv
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import summarise  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def launch_share(path: Path) -> str:
    rows = list(csv.reader(path.open()))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    out = [f"# ncu launch list of one decode step ({sum(v[0] for v in agg.values())} launches, "
           f"{tot / 1e6:.2f} ms summed, cold-cache serialised)\n",
           "| kernel | launches | share of summed time |", "|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {100 * t / tot:.1f}% |")
    return "\n".join(out) + "\n"


def full_report(path: Path) -> str:
    out = [f"# ncu --set full: {path.name}\n"]
    for d in summarise(str(path)):
        out.append(f"## {d.pop('kernel')}\n")
        out.append("| metric | value |\n|---|---|")
        for k, v in d.items():
            out.append(f"| {k} | {v} |")
        out.append("")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    dst = ROOT / "profiles" / rnd
    dst.mkdir(parents=True, exist_ok=True)
    src = ROOT / "gpurun_out"
    if (src / "launches.csv").exists():
        (dst / "launch_share.md").write_text(launch_share(src / "launches.csv"))
    for rep in sorted(src.glob("prof_*.ncu-rep")) + sorted(src.glob("prof_*_raw.csv")):
        tag = rep.name[5:].replace("_raw.csv", "").replace(".ncu-rep", "")
        (dst / f"ncu_{tag}.md").write_text(full_report(rep))
    print("wrote", sorted(p.name for p in dst.iterdir()))
