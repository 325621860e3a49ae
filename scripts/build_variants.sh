#!/bin/bash
# build variant libraries: VARIANTS="name:-DFOO=1 -DBAR=2;name2:..." -> paper_2602_08798_b200/libcgb200_<name>.so
set -e
IFS=';' read -ra VS <<< "${VARIANTS}"
FLAGS=$(python -c "import paper_2602_08798_b200._native as n; print(' '.join(n.NVCC_FLAGS))")
for v in "${VS[@]}"; do
  name=${v%%:*}; defs=${v#*:}
  nvcc $FLAGS $defs -o paper_2602_08798_b200/libcgb200_$name.so paper_2602_08798_b200/csrc/cgb200.cu &
done
wait
ls -la paper_2602_08798_b200/libcgb200_*.so
