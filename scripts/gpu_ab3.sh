#!/bin/bash
# like gpu_ab2.sh plus the NTT microbench per variant
mkdir -p gpurun_out
make -s -C oracle
IFS=';' read -ra VS <<< "${AB}"
for v in "${VS[@]}"; do
  IFS='|' read -r name suf envs <<< "$v"
  lib=paper_2602_08798_b200/libcgb200${suf:+_$suf}.so
  echo "== $name ($lib; $envs)" >> gpurun_out/ab.log
  if [ -z "$NO_PARITY" ]; then
    env CGB_LIB=$lib $envs timeout 900 python -m pytest tests/test_gpu_ring_parity.py tests/test_gpu_primitives.py -q -x 2>&1 | tail -1 >> gpurun_out/ab.log
  fi
  env CGB_LIB=$lib $envs BATCH=216 timeout 300 python scripts/ntt_micro.py 2>/dev/null | python -c "import sys,json; print([(json.loads(l)['dir'], round(json.loads(l)['ns_per_poly'],1)) for l in sys.stdin])" >> gpurun_out/ab.log
  for m in ${KS_MODES:-rotate_add}; do
    env CGB_LIB=$lib KS_MODE=$m $envs timeout 300 python scripts/ks_micro.py 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$m', round(d['us_per_keyswitch'],3), {k:v['ms'] for k,v in d['kernels'].items()})" >> gpurun_out/ab.log
  done
done
cat gpurun_out/ab.log
