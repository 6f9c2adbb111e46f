#!/bin/bash
# Fast A/B builds: the other translation units are compiled once into
# _variants/_obj, then each variant compiles only sim.cu with its -D flags
# (optionally from another source tree: name=DIR:"flags") and links.
#   tools/build_sim_variants.sh new8 "" new4 "-DLA_SIM_WARPS=4 -DLA_SIM_MINB=8"
#   SRC=/tmp/base_wt tools/build_sim_variants.sh base ""
set -e
cd "$(dirname "$0")/.."
ROOT=$(pwd)
SRC=${SRC:-$ROOT}
CS=paper_2208_14567_b200/csrc
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-pthread -I$ROOT/include --expt-relaxed-constexpr"
mkdir -p _variants/_obj
for f in $ROOT/$CS/*.cu $ROOT/$CS/*.cpp; do
  b=$(basename $f); [ "$b" = sim.cu ] && continue
  o=_variants/_obj/$b.o
  if [ ! -f $o ] || [ $f -nt $o ]; then $NV -c $f -o $o & fi
done
wait
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  mkdir -p _variants/$name
  ( $NV $defs -I$ROOT/$CS -c $SRC/$CS/sim.cu -o _variants/$name/sim.o && \
    nvcc -shared -o _variants/$name/liblinks_b200.so _variants/$name/sim.o _variants/_obj/*.o -lcudart && echo built $name ) &
done
wait
