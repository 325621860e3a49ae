#!/bin/bash
# round-end bench lines: headline decode, config 3 (32 tokens), config 2 prefill, config 4 sweep
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
make -s -C oracle
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 900 python bench.py --workload layer --steps 32 > gpurun_out/bench_layer.json 2> gpurun_out/bench_layer.err; echo "layer rc=$?"
timeout 900 python bench.py --workload prefill --steps 1 > gpurun_out/bench_prefill_12h.json 2> gpurun_out/bench_prefill.err; echo "prefill rc=$?"
for LL in 256 512; do
  timeout 600 python bench.py --L $LL --steps 5 --no-cpu-baseline > gpurun_out/bench_decode_L$LL.json 2>/dev/null; echo "L$LL rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
