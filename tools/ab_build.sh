#!/bin/bash
# Build the engine library from the working tree into lib/ab/<name>.so (A/B
# experiments: FHPG_LIB=... python bench.py).
set -e
name=$1
cd "$(dirname "$0")/.."
mkdir -p paper_1208_2428_b200/lib/ab
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude $EXTRA -shared -o paper_1208_2428_b200/lib/ab/$name.so \
  paper_1208_2428_b200/csrc/fhpg_kernels.cu paper_1208_2428_b200/csrc/fhpg_step_fast.cu \
  paper_1208_2428_b200/csrc/fhpg_step_planes.cu paper_1208_2428_b200/csrc/fhpg_step_resident.cu paper_1208_2428_b200/csrc/fhpg_reduce_planes.cu paper_1208_2428_b200/csrc/fhpg_capi.cu \
  paper_1208_2428_b200/csrc/fhpg_tables.cpp
