#!/bin/bash
# full ncu captures of chosen kernels in one decode step: args "regex:skip:count:tag" ...
# Exports raw metrics + per-instruction SASS tables as CSV on the box and keeps the
# .ncu-rep only when small (gpurun copies back <= 64 MiB).
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --profile-step ${BENCH_ARGS:-}"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain.log; exit 1; }
for spec in "$@"; do
  IFS=: read -r rx skip cnt tag <<< "$spec"
  rep=gpurun_out/prof_$tag
  ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_step/" \
      -k regex:$rx -s $skip -c $cnt -o $rep $CMD > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
  ncu -i $rep.ncu-rep --page raw --csv > ${rep}_raw.csv 2>/dev/null
  for ((i = 0; i < cnt; i++)); do
    ncu -i $rep.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 \
        > ${rep}_sass$i.csv 2>/dev/null
  done
  gzip -f ${rep}_sass*.csv
  [ $(stat -c %s $rep.ncu-rep) -gt 20000000 ] && rm -f $rep.ncu-rep
done
du -sh gpurun_out
