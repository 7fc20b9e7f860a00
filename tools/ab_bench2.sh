#!/bin/bash
# Interleaved A/B of lib/ab/*.so variants on cfg4 without and with forcing
# (GPU box): bash tools/ab_bench2.sh v1 v2 ... -> gpurun_out/ab2.txt
cd "$(dirname "$0")/.."
for round in 1 2; do
  for v in "$@"; do
    a=$(FHPG_LIB=$PWD/paper_1208_2428_b200/lib/ab/$v.so timeout 300 python tools/ab_time.py 16384 16384 fhp3 0 100 2>/dev/null | tail -1)
    b=$(FHPG_LIB=$PWD/paper_1208_2428_b200/lib/ab/$v.so timeout 300 python tools/ab_time.py 16384 16384 fhp3 0.01 50 2>/dev/null | tail -1)
    echo "$v round$round p0=$a p001=$b" | tee -a gpurun_out/ab2.txt
  done
done
