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
bash scripts/gpu_ncu.sh ${NCU_SPECS:-"k_ks_row:20:1:ks_row" "k_col_fused:20:2:col_fused" "k_ntt2_fpr:40:2:ntt2_fpr"}
