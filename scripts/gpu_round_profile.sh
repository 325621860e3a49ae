#!/bin/bash
# round deliverable: full bench line, ncu launch list of one step, ncu --set full of the top kernels
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
make -s -C oracle
python bench.py --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --profile-step"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
bash scripts/gpu_ncu.sh ${NCU_SPECS:-"k_ks_row:40:2:ks_row" "k_col_fused:20:2:col_fused" "k_ntt2_fpr:40:2:ntt2_fpr"}
# config 3 (decoder layer) and configs 2 / 4 bench lines
python bench.py --workload layer --steps 32 > gpurun_out/bench_layer.json 2> gpurun_out/bench_layer.err
echo "layer rc=$?"
python bench.py --workload prefill --steps 1 > gpurun_out/bench_prefill_12h.json 2> gpurun_out/bench_prefill.err
python bench.py --L 256 --steps 5 --no-cpu-baseline > gpurun_out/bench_decode_L256.json 2>/dev/null
python bench.py --L 512 --steps 5 --no-cpu-baseline > gpurun_out/bench_decode_L512.json 2>/dev/null
echo "configs rc=$?"
