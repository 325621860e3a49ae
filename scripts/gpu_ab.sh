#!/bin/bash
# A/B of an env toggle on the decode bench: ENVS="CGB_FP_REGIO=0;CGB_FP_REGIO=1"
set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_primitives.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/ab_tests.log
IFS=';' read -ra VARIANTS <<< "${ENVS}"
for v in "${VARIANTS[@]}"; do
  for rep in 1 2; do
    echo "== $v rep $rep" >> gpurun_out/ab.log
    env $v timeout 300 python bench.py --steps ${STEPS:-6} --warmup 3 --no-cpu-baseline 2>>gpurun_out/ab.err | tail -1 >> gpurun_out/ab.log
  done
done
