#!/bin/bash
# Fast A/B builds of one translation unit (FILE=chamfer.cu, default sim.cu):
# the other units are compiled once into _variants/_obj_$FILE, each variant
# compiles only FILE with its -D flags and links.
#   FILE=chamfer.cu tools/build_file_variants.sh s32 "-DLA_CH_INDEX_SEED_DIV=32" s128 "-DLA_CH_INDEX_SEED_DIV=128"
set -e
cd "$(dirname "$0")/.."
ROOT=$(pwd)
FILE=${FILE:-sim.cu}
CS=paper_2208_14567_b200/csrc
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-pthread -I$ROOT/include --expt-relaxed-constexpr"
OBJ=_variants/_obj_$FILE
mkdir -p $OBJ
for f in $ROOT/$CS/*.cu $ROOT/$CS/*.cpp; do
  b=$(basename $f); [ "$b" = "$FILE" ] && continue
  o=$OBJ/$b.o
  if [ ! -f $o ] || [ $f -nt $o ]; then $NV -c $f -o $o & fi
done
wait
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  mkdir -p _variants/$name
  ( $NV $defs -I$ROOT/$CS -c $ROOT/$CS/$FILE -o _variants/$name/unit.o && \
    nvcc -shared -o _variants/$name/liblinks_b200.so _variants/$name/unit.o $OBJ/*.o -lcudart && echo built $name ) &
done
wait
