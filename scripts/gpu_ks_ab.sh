#!/bin/bash
# A/B of key-switch library variants (paper_2602_08798_b200/libcgb200_<v>.so):
# word parity on the benchmarked ring, key-switch microbench, decode bench
mkdir -p gpurun_out
make -s -C oracle
for v in ${VARIANTS_AB}; do
  lib=paper_2602_08798_b200/libcgb200_$v.so
  echo "== $v" >> gpurun_out/ab.log
  CGB_LIB=$lib timeout 600 python -m pytest tests/test_gpu_ring_parity.py -q -x -k "rotate or attention" 2>&1 | tail -1 >> gpurun_out/ab.log
  for m in rotate_add distinct; do
    CGB_LIB=$lib KS_MODE=$m timeout 300 python scripts/ks_micro.py 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$m', round(d['us_per_keyswitch'],3), {k:v['ms'] for k,v in d['kernels'].items()})" >> gpurun_out/ab.log
  done
  for rep in 1 2; do
    CGB_LIB=$lib timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('bench', round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], {k:v['ms'] for k,v in list(d['kernels'].items())[:6]})" >> gpurun_out/ab.log
  done
done
cat gpurun_out/ab.log
