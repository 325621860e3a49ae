#!/bin/bash
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q -x -rfE > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
for e in "CGB_EXT_A=0" "CGB_EXT_A=1"; do for rep in 1 2; do
env $e timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$e', round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], {k:v['ms'] for k,v in list(d['units'].items())[:3]}, {k:d['kernels'][k]['ms'] for k in ('scale_round','lift_QB','tensor','ntt_inv','ntt_fwd') if k in d['kernels']})"
done; done
