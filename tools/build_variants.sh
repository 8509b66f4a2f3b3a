#!/bin/bash
# Build libpt variants for A/B timing from the archived round-1 exhaustive.cu (every
# rejected kernel variant, selected by -D flags):
#   tools/build_variants.sh name "-DX=1 -DY=2" ...   ->  variants/libpt_<name>.so  (use with PT_LIB=...)
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
SRCS=$(ls paper_2507_15277_b200/csrc/*.cu | grep -v '/exhaustive.cu$')
while [ $# -ge 2 ]; do
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    -Iinclude -Ipaper_2507_15277_b200/csrc --expt-relaxed-constexpr $2 -shared -o variants/libpt_$1.so \
    $SRCS tools/r1_variants/exhaustive_variants.cu -ldl &
  shift 2
done
wait
