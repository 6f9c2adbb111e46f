#!/bin/bash
# Round-2 GPU pass (one B200): tests, smoke, bench + reference arm, launch
# list of the C2 step, per-kernel metrics table, --set full captures of the
# top kernels (C2 screen + write, C4 pruned scan, C5 multi-query scan, C3
# gate).  Outputs in gpurun_out/r02_*; summarise into profiles/.
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/r02_gputests.log 2>&1; echo "tests rc=$?" >> $O/r02_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r02_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r02_smoke.log
timeout 1200 python bench.py > $O/r02_bench.log 2>&1; echo "bench rc=$?" >> $O/r02_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/r02_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches.csv \
  python bench.py --steps 2 --warmup 3 --skip c1,c3,c4,c5,gen,cpu > $O/r02_ncu_launch.log 2>&1
M=$(python -c "import sys; sys.path.insert(0, 'tools'); import ncu_table; print(','.join(ncu_table.METRICS))")
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file $O/r02_table.csv python tools/kernel_table.py \
  > $O/r02_ncu_table.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -c 2 -f -o $O/r02_c2 \
  python tools/profile_step.py c2 1 > $O/r02_ncu_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chamfer_scan --launch-skip 2 -c 1 -f \
  -o $O/r02_c4 python tools/time_prune.py > $O/r02_ncu_c4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:index_bound -c 1 -f \
  -o $O/r02_c4_index python tools/time_index.py --once > $O/r02_ncu_c4_index.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches_c4.csv \
  python tools/time_index.py --once > $O/r02_ncu_launch_c4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chamfer_mq --launch-skip 1 -c 1 -f \
  -o $O/r02_c5 python tools/profile_c5chamfer.py > $O/r02_ncu_c5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sim_kernel --launch-skip 1 -c 1 -f \
  -o $O/r02_c3 python tools/time_c3.py 2000000 > $O/r02_ncu_c3.log 2>&1
# summaries on the box; the reports themselves (tens of MB each with sources)
# stay behind unless KEEP_REPS is set (gpurun returns at most 64 MiB)
for n in c2 c3 c4 c4_index c5; do
  python tools/ncu_summary.py $O/r02_$n.ncu-rep > $O/r02_ncu_$n.txt 2>&1
  python tools/ncu_lines.py $O/r02_$n.ncu-rep 0 40 > $O/r02_lines_$n.txt 2>&1
  [ -n "$KEEP_REPS" ] || rm -f $O/r02_$n.ncu-rep
done
python tools/launch_list.py $O/r02_launches.csv > $O/r02_launch_list_c2.txt 2>&1
python tools/launch_list.py $O/r02_launches_c4.csv > $O/r02_launch_list_c4.txt 2>&1
python tools/ncu_table.py $O/r02_table.csv > $O/r02_kernel_table.txt 2>&1
du -sh $O
echo done
