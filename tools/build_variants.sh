#!/bin/bash
# Build liblinks_b200.so variants of the fp32-screen error model for sweeps:
#   tools/build_variants.sh name "-DLA_ERR_STEP=5e-7f -DLA_MARGIN_K=3.0f" ...
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  mkdir -p ${VDIR:-tools/_variants}/$name
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-pthread -shared \
    -Iinclude --expt-relaxed-constexpr $defs -o ${VDIR:-tools/_variants}/$name/liblinks_b200.so \
    paper_2208_14567_b200/csrc/*.cu paper_2208_14567_b200/csrc/*.cpp -lcudart &
done
wait
