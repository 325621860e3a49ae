#!/bin/bash
# key-switch microbench + one ncu --set full capture of one batched key switch (5 launches)
mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
TAG=${TAG:-ks}
python scripts/ks_micro.py > gpurun_out/${TAG}_micro.json 2> gpurun_out/${TAG}_micro.err
echo "micro rc=$?"; cat gpurun_out/${TAG}_micro.json
if [ -z "$NO_NCU" ]; then
KS_PROFILE=1 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ks/" \
  -o gpurun_out/prof_${TAG} python scripts/ks_micro.py > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
n=$(ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv 2>/dev/null | tail -n +3 | wc -l)
for ((i = 0; i < n; i++)); do
  ncu -i gpurun_out/prof_${TAG}.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 \
      > gpurun_out/prof_${TAG}_sass$i.csv 2>/dev/null
done
gzip -f gpurun_out/prof_${TAG}_sass*.csv
[ $(stat -c %s gpurun_out/prof_${TAG}.ncu-rep) -gt 30000000 ] && rm -f gpurun_out/prof_${TAG}.ncu-rep
fi
du -sh gpurun_out
