#!/bin/bash
# launch list of one decode step + full ncu capture of the top kernel
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --profile-step"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_step/" \
    -k regex:${KERNEL:-k_ntt} -c ${COUNT:-3} -o gpurun_out/prof_${TAG:-ntt} $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -5 gpurun_out/ncu_full.log
