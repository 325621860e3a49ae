#!/bin/bash
# GPU tests, then the decoder-layer bench with / without the rotation dedup + hoisted key switch
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build(verbose=True)" > gpurun_out/build.log 2>&1
make -s -C oracle
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 | tee gpurun_out/pytest_gpu.log
for v in "0 0" "1 0" "1 1"; do
  set -- $v
  CGB_ROT_DEDUP=$1 CGB_KS_HOIST=$2 timeout 600 python bench.py --workload layer --steps ${LSTEPS:-8} --warmup 3 --no-cpu-baseline \
    2>> gpurun_out/layer.err | tail -1 > gpurun_out/layer_dedup$1_hoist$2.json
  echo "dedup=$1 hoist=$2 rc=$?"; python -c "import json,sys; d=json.load(open('gpurun_out/layer_dedup$1_hoist$2.json')); print(d['value'], d['prefill_ms'], d['tokens'][:8], d['gpu_launches'])"
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print('decode', d['value'], d['e2e']['value'], d['roofline']['frac'])"
