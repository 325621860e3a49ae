#!/bin/bash
# hoisted key switch: microbenchmark, ncu capture of k_ks_inner_hoist, then the
# round's bench lines (headline decode, config 3 layer over 32 tokens)
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/hoist_micro.py > gpurun_out/hoist_micro.json 2> gpurun_out/hoist_micro.err
echo "micro rc=$?"
HOIST_K=64 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ks_inner_hoist -s 2 -c 1 \
  -o gpurun_out/prof_hoist python scripts/hoist_micro.py > gpurun_out/ncu_hoist.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_hoist.ncu-rep --page raw --csv > gpurun_out/prof_hoist_raw.csv 2>/dev/null
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?"
timeout 900 python bench.py --workload layer --steps 32 > gpurun_out/bench_layer.json 2> gpurun_out/bench_layer.err
echo "layer rc=$?"
