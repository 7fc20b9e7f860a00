#!/bin/bash
# Interleaved bench of lib/ab/*.so variants (run on the GPU box):
#   bash tools/ab_bench.sh v1 v2 ...   -> gpurun_out/ab.txt
cd "$(dirname "$0")/.."
for round in 1 2; do
  for v in "$@"; do
    val=$(FHPG_LIB=$PWD/paper_1208_2428_b200/lib/ab/$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 100 --warmup 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'])")
    echo "$v round$round $val" | tee -a gpurun_out/ab.txt
  done
done
