#!/bin/bash
# round 2: GPU test suite (incl. the word-parity and drop-in suites), then one bench line
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
make -s -C oracle
export CGB_REF_SUITE_OUT=gpurun_out/ref_suite.json
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -rfE --durations=20 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ('value','e2e','roofline','units','clocks')})"
fi
