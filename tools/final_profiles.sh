#!/bin/bash
# Round-end GPU pass (one B200): tests, smoke, bench, launch list, per-kernel
# metrics table and --set full captures of the top kernels.  Outputs in
# gpurun_out/; summarise into profiles/ with tools/ncu_summary.py and
# tools/ncu_table.py.
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/final_gputests.log 2>&1; echo "tests rc=$?" >> $O/final_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1; echo "smoke rc=$?" >> $O/final_smoke.log
timeout 900 python bench.py > $O/final_bench.log 2>&1; echo "bench rc=$?" >> $O/final_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/final_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/final_launches.csv \
  python bench.py --steps 2 --warmup 3 --skip c3,c4,c5,gen,cpu > $O/final_ncu_launch.log 2>&1
M=$(python -c "import sys; sys.path.insert(0, 'tools'); import ncu_table; print(','.join(ncu_table.METRICS))")
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file $O/final_table.csv python tools/kernel_table.py \
  > $O/final_ncu_table.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -c 2 -f -o $O/final_c2 \
  python tools/profile_step.py c2 1 > $O/final_ncu_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chamfer_scan -c 1 -f -o $O/final_c4 \
  python tools/profile_step.py c4 1 > $O/final_ncu_c4.log 2>&1
echo done
