"""Print value / e2e / idle and the top kernels of each bench line in gpurun_out/ab.log."""
import json
for line in open("gpurun_out/ab.log"):
    if line.startswith("=="):
        print(line.strip())
        continue
    try:
        d = json.loads(line)
    except Exception:
        print("  ?", line[:160])
        continue
    ks = sorted(d["kernels"].items(), key=lambda kv: -kv[1]["ms"])[:5]
    print("  value %.2f e2e %.2f idle %s | %s" % (d["value"], d["e2e"]["value"], d.get("gpu_idle_ms_per_step"),
          ", ".join("%s %.1f" % (k, v["ms"]) for k, v in ks)))
