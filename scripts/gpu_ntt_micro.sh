#!/bin/bash
# NTT variants A/B (ENVS="A=1;A=0"), then optional ncu of NCU_KERNEL under NCU_ENV
mkdir -p gpurun_out
IFS=';' read -ra VARIANTS <<< "${ENVS}"
for v in "${VARIANTS[@]}"; do
  env $v VARIANT="$v" timeout 120 python scripts/ntt_micro.py >> gpurun_out/ntt_micro.log 2>>gpurun_out/ntt_micro.err
done
if [ -n "${NCU_KERNEL:-}" ]; then
  env ${NCU_ENV:-} ITERS=2 BATCH=36 timeout 600 ncu --set full --clock-control none --import-source on \
    -k "regex:${NCU_KERNEL}" -c ${NCU_COUNT:-4} -o gpurun_out/${NCU_OUT:-ntt_micro} -f \
    python scripts/ntt_micro.py > gpurun_out/ncu_micro.log 2>&1
  echo "ncu rc=$?"
fi
