"""A/B of the validity screen: warp-per-candidate kernel (default, lanes =
angles) vs the lane-per-candidate kernel (LA_SIM_LANE_SCREEN), on the C2 deferred screen
(100k 6-8 joint candidates) and the C3 gate (5-20 joints padded to 20).
Prints times, work counters and flag mismatches between the two kernels.

    python tools/time_screen.py [c3_count] [refill,replay ...]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_14567_b200 import _native as N  # noqa: E402
from paper_2208_14567_b200.solver import simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import mixed_batch, native_batch  # noqa: E402

C3N = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
PARAMS = [tuple(int(v) for v in a.split(",")) for a in sys.argv[2:]] or [(0, 0)]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def run(name, pos, table, topo, **kw):
    outs = {}
    for label, extra, scr in [("warp", 0, (0, 0))] + [(f"lane{p}", N.LA_SIM_LANE_SCREEN, p) for p in PARAMS]:
        def f():
            outs[label] = simulate_tensors(pos, table, 200, topo, write_traj=False, low=True,
                                           _extra_flags=extra | kw.get("flags", 0), _screen=scr,
                                           gate_only=kw.get("gate_only", False))
        ms = timed(f)
        c = torch.zeros(8, dtype=torch.int64, device="cuda")
        simulate_tensors(pos, table, 200, topo, write_traj=False, low=True, counters=c,
                         _extra_flags=extra | kw.get("flags", 0), _screen=scr, gate_only=kw.get("gate_only", False))
        c = c.cpu().numpy()
        print(f"{name} {label:12s} {ms:8.3f} ms  replays {c[0]:>10d} slots {c[1]:>11d} dyad-slots {c[2]:>12d} "
              f"cand {c[3]:>9d} events {c[4]:>8d} lane-angles {c[5]:>11d} dyads {c[6]:>12d}", flush=True)
    ref = outs["warp"]
    for label, o in outs.items():
        if label == "warp":
            continue
        mm = {k: int((o[k] != ref[k]).sum().item()) for k in ("first_t", "first_joint", "low_t", "low_joint")}
        print(f"{name} {label} mismatches vs warp: {mm}", flush=True)


mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
run("C2-defer", torch.from_numpy(mb.pos).cuda(), mb.table(), torch.from_numpy(mb.topo).cuda(), flags=N.LA_SIM_DEFER)
run("C2-full ", torch.from_numpy(mb.pos).cuda(), mb.table(), torch.from_numpy(mb.topo).cuda())
nb = native_batch(C3N, 5, 20, seed=3000)
run("C3-gate ", torch.from_numpy(nb.pos).cuda(), nb.table, torch.from_numpy(nb.topo).cuda(), gate_only=True)
