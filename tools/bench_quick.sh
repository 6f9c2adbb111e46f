#!/bin/bash
# quick GPU check: gpu tests + bench summary
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gputests.log
timeout 500 python bench.py --steps 5 --warmup 3 --skip cpu ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
print("C2 sims/s %.3e" % d["value"], {k: round(v, 4) for k, v in d["kernels_ms"].items()}, "e2e %.3e" % d["e2e"]["value"])
print([(r["kernel"], round(r["frac"], 3)) for r in d["roofline_kernels"]], d["clocks"])
s = d["secondary"]
if "screen" in s:
    print("C3 cand/s %.3e frac %.3f fixups %.4f" % (s["screen"]["value"], s["screen"]["roofline"]["frac"], s["screen"]["fixup_lane_angles"] / s["screen"]["angles_evaluated"]))
if "end_to_end" in s:
    e = s["end_to_end"]
    print("C5 cand/s %.3e" % e["value"], {k: round(v, 3) for k, v in e["stages_ms"].items()}, "valid", e["valid_per_gpu"], "curves", e["curves_per_gpu"], "norm frac %.3f" % e["normalize"]["frac_fp32"], "chamfer pairs/s %.3e" % e["chamfer"]["pairs/s"])
if "chamfer" in s:
    print("C4 pairs/s %.3e frac %.3f" % (s["chamfer"]["value"], s["chamfer"]["roofline"]["frac"]))
PY
