#!/bin/bash
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
make -s -C oracle
timeout 1200 python -m pytest tests/test_gpu_primitives.py -q -rfE --durations=8 > gpurun_out/pytest_prim.log 2>&1
echo "prim rc=$?"; tail -12 gpurun_out/pytest_prim.log
timeout 1500 python bench_kernels.py > gpurun_out/kernels_c5.jsonl 2> gpurun_out/kernels_c5.err
echo "c5 rc=$?"; tail -3 gpurun_out/kernels_c5.err
python - <<'PY'
import json
for l in open('gpurun_out/kernels_c5.jsonl'):
    d=json.loads(l)
    if d['kernel'] in ('keyswitch_rotate','mult_cipher','ntt_fwd'):
        print(d['kernel'], d['logN'], d['limbs'], round(d.get('us_per_ct', d['ms']),3), round(d.get('modmul_pipe_frac') or 0,3), round(d['hbm_frac'],3), d['clocks']['sm_mhz'])
PY
