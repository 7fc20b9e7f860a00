#!/bin/bash
# ncu --set full of one step_ring launch for each lib/ab/<variant>.so (GPU box):
#   bash tools/ncu_ab.sh v1 v2 ...   -> gpurun_out/ncu_<v>.ncu-rep (+ raw csv)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  FHPG_LIB=$PWD/paper_1208_2428_b200/lib/ab/$v.so timeout 600 ncu --set full --import-source on \
    --clock-control none -k regex:"step_(ring|pair)" -s 2 -c 1 -o gpurun_out/ncu_$v -f \
    python tools/profile_step.py 4 > gpurun_out/ncu_$v.log 2>&1
  echo "$v ncu=$?"
  ncu -i gpurun_out/ncu_$v.ncu-rep --page raw --csv > gpurun_out/ncu_${v}_raw.csv 2>/dev/null
  ncu -i gpurun_out/ncu_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${v}_sass.csv 2>/dev/null
done
