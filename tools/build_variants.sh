#!/bin/bash
# build libpt variants with -D flags for A/B timing: tools/build_variants.sh name "-DX=1 -DY=2" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -ge 2 ]; do
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    -Iinclude --expt-relaxed-constexpr $2 -shared -o variants/libpt_$1.so paper_2507_15277_b200/csrc/*.cu &
  shift 2
done
wait
