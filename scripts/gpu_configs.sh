#!/bin/bash
# noise margins of the default rings + bench lines for configs 2 (prefill) and 4 (L sweep)
mkdir -p gpurun_out
for L in 3 4; do CGB_LIMBS=$L timeout 600 python scripts/noise_probe.py >> gpurun_out/noise.jsonl 2>> gpurun_out/noise.err; done
for LL in 256 512; do
  timeout 900 python bench.py --L $LL --steps 5 --warmup 3 --no-cpu-baseline 2>> gpurun_out/cfg.err | tail -1 > gpurun_out/bench_L$LL.json
done
timeout 1500 python bench.py --workload prefill --steps 1 --warmup 3 --no-cpu-baseline 2>> gpurun_out/cfg.err | tail -1 > gpurun_out/bench_prefill.json
