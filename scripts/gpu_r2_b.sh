#!/bin/bash
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q -rfE --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload prefill --steps 1 > gpurun_out/bench_prefill.json 2> gpurun_out/bench_prefill.err
echo "prefill rc=$?"; tail -c 1500 gpurun_out/bench_prefill.json; tail -3 gpurun_out/bench_prefill.err
timeout 1200 python bench.py --workload layer --steps 8 > gpurun_out/bench_layer.json 2> gpurun_out/bench_layer.err
echo "layer rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bench_layer.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ('value','steady_state_ms_per_token','prefill_ms','clocks','cpu_baseline')}, d['roofline']['frac'])"; tail -3 gpurun_out/bench_layer.err
