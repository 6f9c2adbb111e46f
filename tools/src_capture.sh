#!/bin/bash
# ncu capture of the C2 step kernels with per-source-line counters (and the
# C3 gate screen); read with tools/src_lines.py
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 300 python tools/counters_c2.py > $O/counters_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -c 2 -f -o $O/src_c2 \
  python tools/profile_step.py c2 1 > $O/src_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sim_kernel --launch-skip 1 -c 1 -f \
  -o $O/src_c3 python tools/time_c3.py 2000000 > $O/src_c3.log 2>&1
echo done
