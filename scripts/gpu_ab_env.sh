#!/bin/bash
# parity subset + decode bench A/B over environment settings: ENVS="A=0;A=1"
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
make -s -C oracle
timeout 1200 python -m pytest tests/test_gpu_ring_parity.py tests/test_gpu_primitives.py tests/test_gpu_hotpath.py -q -x ${PYTEST_K} 2>&1 | tail -2
IFS=';' read -ra VS <<< "${ENVS}"
for e in "${VS[@]}"; do for rep in 1 2; do
env $e timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$e', round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], {k:v['ms'] for k,v in list(d['units'].items())[:4]}, {k:d['kernels'][k]['ms'] for k in ('scale_round','tensor','tensor_intt','ntt_inv','ntt_fwd') if k in d['kernels']})"
done; done
if [ -n "$PREFILL" ]; then for e in "${VS[@]}"; do
env $e timeout 600 python bench.py --workload prefill --steps 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('prefill $e', round(d['value'],1), {k:v['ms'] for k,v in list(d['units'].items())[:4]})"
done; fi
