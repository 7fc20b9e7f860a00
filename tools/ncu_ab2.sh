#!/bin/bash
# As ncu_ab.sh, without ncu's cache flush between replays (--cache-control none):
#   bash tools/ncu_ab2.sh v1 v2 ...  -> gpurun_out/ncu2_<v>_raw.csv
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  FHPG_LIB=$PWD/paper_1208_2428_b200/lib/ab/$v.so timeout 600 ncu --set full --import-source on \
    --clock-control none --cache-control none -k regex:"step_ring" -s 6 -c 1 -o gpurun_out/ncu2_$v -f \
    python tools/profile_step.py 8 > gpurun_out/ncu2_$v.log 2>&1
  echo "$v ncu=$?"
  ncu -i gpurun_out/ncu2_$v.ncu-rep --page raw --csv > gpurun_out/ncu2_${v}_raw.csv 2>/dev/null
  ncu -i gpurun_out/ncu2_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu2_${v}_sass.csv 2>/dev/null
done
