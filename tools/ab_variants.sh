#!/bin/bash
# A/B of library variants on one GPU box: for each variant dir under
# _variants/, install its liblinks_b200.so in place and run the given command.
#   bash tools/ab_variants.sh "python tools/time_prune.py" head d1 d2
cd "$(dirname "$0")/.."
cmd=$1; shift
cp paper_2208_14567_b200/_lib/liblinks_b200.so /tmp/_cur_lib.so
for v in "$@"; do
  cp _variants/$v/liblinks_b200.so paper_2208_14567_b200/_lib/liblinks_b200.so
  echo "== $v"; eval "$cmd"
done
cp /tmp/_cur_lib.so paper_2208_14567_b200/_lib/liblinks_b200.so
