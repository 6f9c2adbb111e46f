#!/bin/bash
# Quick GPU pass: GPU tests, smoke, bench (ours + reference arm).
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/p1_gputests.log 2>&1; echo "tests rc=$?" >> $O/p1_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/p1_smoke.log 2>&1; echo "smoke rc=$?" >> $O/p1_smoke.log
timeout 1200 python bench.py > $O/p1_bench.log 2>&1; echo "bench rc=$?" >> $O/p1_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/p1_bench_ref.log 2>&1; echo "ref rc=$?" >> $O/p1_bench_ref.log
echo done
