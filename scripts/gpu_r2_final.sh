#!/bin/bash
# round-2 deliverables: GPU tests, decode bench (L = 128 / 256 / 512), prefill, layer, ncu launch list
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
make -s -C oracle
if [ -z "$NO_TESTS" ]; then
  CGB_REF_SUITE_OUT=gpurun_out/ref_suite.json timeout 1500 python -m pytest tests -m gpu -q -rfE > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
fi
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_arm.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?"
for L in 256 512; do
  timeout 600 python bench.py --L $L --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_decode_L$L.json 2>/dev/null
done
timeout 900 python bench.py --workload prefill --steps 1 > gpurun_out/bench_prefill_12h.json 2> gpurun_out/bench_prefill.err
echo "prefill rc=$?"
timeout 1500 python bench.py --workload layer --steps 8 > gpurun_out/bench_layer.json 2> gpurun_out/bench_layer.err
echo "layer rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --profile-step --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
python - <<'PY'
import json
for f in ("bench_full","bench_decode_L256","bench_decode_L512","bench_prefill_12h","bench_layer","bench_reference_arm"):
    try:
        d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("e2e",{}).get("value"), (d.get("clocks") or {}).get("sm_mhz"), (d.get("roofline") or {}).get("frac"), (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e: print(f, "ERR", e)
PY
