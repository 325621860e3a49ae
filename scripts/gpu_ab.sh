#!/bin/bash
# GPU tests under each PARITY_ENVS variant, then decode bench A/B: ENVS="A=0;A=1"
set -u
mkdir -p gpurun_out
IFS=';' read -ra PV <<< "${PARITY_ENVS:-X=0}"
for v in "${PV[@]}"; do
  echo "== $v" >> gpurun_out/ab_tests.log
  env $v timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/ab_tests.log
done
IFS=';' read -ra VARIANTS <<< "${ENVS}"
for v in "${VARIANTS[@]}"; do
  for rep in 1 2; do
    echo "== $v rep $rep" >> gpurun_out/ab.log
    env $v timeout 300 python bench.py --steps ${STEPS:-6} --warmup 3 --no-cpu-baseline 2>>gpurun_out/ab.err | tail -1 >> gpurun_out/ab.log
  done
done
