#!/bin/bash
# Build the engine library from the working tree into lib/ab/<name>.so (A/B
# experiments: FHPG_LIB=... python bench.py). Extra nvcc flags in $EXTRA
# (e.g. EXTRA="-DFHPG_WAIT_HINT=100000"); the translation units compile in
# parallel.
set -e
name=$1
cd "$(dirname "$0")/.."
out=paper_1208_2428_b200/lib/ab
obj=/tmp/ab_obj_$name
mkdir -p $out $obj
flags="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude $EXTRA"
pids=()
for f in fhpg_kernels.cu fhpg_step_fast.cu fhpg_step_planes.cu fhpg_step_resident.cu \
         fhpg_reduce_planes.cu fhpg_capi.cu fhpg_tables.cpp; do
  /usr/local/cuda/bin/nvcc $flags -c -o $obj/$f.o paper_1208_2428_b200/csrc/$f &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/$name.so $obj/*.o
echo built $out/$name.so
