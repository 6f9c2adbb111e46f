#!/bin/bash
# One-B200 pass: GPU tests, smoke, bench (+ reference arm), launch lists of
# the C2 step and the pruned C4 scan, --set full capture of the pruned scan.
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/rp_gputests.log 2>&1; echo "tests rc=$?" >> $O/rp_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/rp_smoke.log 2>&1; echo "smoke rc=$?" >> $O/rp_smoke.log
timeout 900 python bench.py > $O/rp_bench.log 2>&1; echo "bench rc=$?" >> $O/rp_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/rp_bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/rp_launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --skip c3,c4,c5,gen,cpu > $O/rp_ncu_launch_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:chamfer|lb_grid|thr_init|merge_kernel' \
  --csv --log-file $O/rp_launches_c4.csv python tools/time_prune.py > $O/rp_ncu_launch_c4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chamfer_scan --launch-skip 2 -c 1 -f \
  -o $O/rp_c4_pruned python tools/time_prune.py > $O/rp_ncu_c4.log 2>&1
echo done
