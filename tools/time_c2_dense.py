"""C2 deferred pipeline: strided vs dense path rows (A/B in one process)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.solver import simulate_deferred  # noqa: E402
from paper_2208_14567_b200.workloads import mixed_batch  # noqa: E402

mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
pos = torch.from_numpy(mb.pos).cuda()
topo = torch.from_numpy(mb.topo).cuda()
table = mb.table()
traj = torch.empty((mb.B * 8, 200, 2), dtype=torch.float32, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


class Tm:
    def __init__(self):
        self.ev = []

    def mark(self, n):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev.append((n, e))


for dense in (False, True, False, True):
    for _ in range(3):
        simulate_deferred(pos, table, 200, topo, traj=traj, dense_rows=dense)
    agg = {}
    for _ in range(20):
        flush.zero_()
        t = Tm()
        t.mark("start")
        simulate_deferred(pos, table, 200, topo, traj=traj, timer=t, dense_rows=dense)
        t.mark("end")
        torch.cuda.synchronize()
        for (n0, e0), (n1, e1) in zip(t.ev, t.ev[1:]):
            agg.setdefault(n1, []).append(e0.elapsed_time(e1))
    print("dense" if dense else "strided", {k: round(statistics.median(v), 4) for k, v in agg.items()},
          "total", round(sum(statistics.median(v) for v in agg.values()), 4), flush=True)
