#!/bin/bash
# NTT iteration: parity tests under each PARITY_ENVS variant, microbench A/B, optional ncu
mkdir -p gpurun_out
IFS=';' read -ra PV <<< "${PARITY_ENVS:-X=0}"
for v in "${PV[@]}"; do
  echo "== $v" >> gpurun_out/ntt_parity.log
  env $v timeout 300 python -m pytest tests/test_gpu_primitives.py -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/ntt_parity.log
done
bash scripts/gpu_ntt_micro.sh
