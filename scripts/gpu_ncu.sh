#!/bin/bash
# full ncu captures of chosen kernels in one decode step: args "regex:skip:count:tag" ...
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --profile-step"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain.log; exit 1; }
for spec in "$@"; do
  IFS=: read -r rx skip cnt tag <<< "$spec"
  ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_step/" \
      -k regex:$rx -s $skip -c $cnt -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
done
