#!/bin/bash
# one GPU box call: build, GPU parity tests, a short bench run
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build(verbose=True)" > gpurun_out/build.log 2>&1
make -s -C oracle
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -40 | tee gpurun_out/pytest_gpu.log
timeout ${BENCH_TIMEOUT:-600} python bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-3} ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.json; tail -20 gpurun_out/bench.err
