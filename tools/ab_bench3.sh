#!/bin/bash
# Interleaved A/B of lib/ab/*.so variants (GPU box): cfg4 FHP-III p = 0,
# p = 0.01 and the reference's DEFAULT table, 2 rounds -> gpurun_out/ab3.txt
#   bash tools/ab_bench3.sh v1 v2 ...
cd "$(dirname "$0")/.."
for round in 1 2; do
  for v in "$@"; do
    L=$PWD/paper_1208_2428_b200/lib/ab/$v.so
    a=$(FHPG_LIB=$L timeout 300 python tools/ab_time.py 16384 16384 fhp3 0 100 2>/dev/null | tail -1)
    b=$(FHPG_LIB=$L timeout 300 python tools/ab_time.py 16384 16384 fhp3 0.01 50 2>/dev/null | tail -1)
    c=$(FHPG_LIB=$L timeout 300 python tools/ab_time.py 16384 16384 default 0 100 2>/dev/null | tail -1)
    echo "$v round$round p0=$a p001=$b default=$c" | tee -a gpurun_out/ab3.txt
  done
done
