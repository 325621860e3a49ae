#!/bin/bash
# A/B of key-switch variants.  AB="name|libsuffix|ENV=1 ENV2=2;name2||..." (libsuffix empty: the default library).
# Per variant: word parity on the benchmarked ring (rotate tests), key-switch microbench (per-kernel ms),
# optionally (BENCH=1) two decode bench runs.
mkdir -p gpurun_out
make -s -C oracle
IFS=';' read -ra VS <<< "${AB}"
for v in "${VS[@]}"; do
  IFS='|' read -r name suf envs <<< "$v"
  lib=paper_2602_08798_b200/libcgb200${suf:+_$suf}.so
  echo "== $name ($lib; $envs)" >> gpurun_out/ab.log
  if [ -z "$NO_PARITY" ]; then
    env CGB_LIB=$lib $envs timeout 600 python -m pytest tests/test_gpu_ring_parity.py -q -x -k "${PARITY_K:-rotate}" 2>&1 | tail -1 >> gpurun_out/ab.log
  fi
  for m in ${KS_MODES:-rotate_add}; do
    env CGB_LIB=$lib KS_MODE=$m $envs timeout 300 python scripts/ks_micro.py 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$m', round(d['us_per_keyswitch'],3), {k:v['ms'] for k,v in d['kernels'].items()})" >> gpurun_out/ab.log
  done
  if [ -n "$BENCH" ]; then
    for rep in 1 2; do
      env CGB_LIB=$lib $envs timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('bench', round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], {k:v['ms'] for k,v in list(d['units'].items())[:4]})" >> gpurun_out/ab.log
    done
  fi
done
cat gpurun_out/ab.log
