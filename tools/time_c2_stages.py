"""Per-stage times of the C2 deferred pipeline (screen / paths / compact), median of 10."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.solver import simulate_deferred  # noqa: E402
from paper_2208_14567_b200.workloads import mixed_batch  # noqa: E402

mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
pos, topo, table = torch.from_numpy(mb.pos).cuda(), torch.from_numpy(mb.topo).cuda(), mb.table()
traj = torch.empty((mb.B * 8, 200, 2), dtype=torch.float32, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


class T:
    def __init__(self):
        self.ev = [("start", torch.cuda.Event(enable_timing=True))]
        self.ev[0][1].record()

    def mark(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev.append((name, e))


res = {}
for i in range(13):
    flush.zero_()
    t = T()
    simulate_deferred(pos, table, 200, topo, traj=traj, dense_rows=True, timer=t,
                      split_rows="split" in sys.argv)
    torch.cuda.synchronize()
    if i >= 3:
        for (a, ea), (b, eb) in zip(t.ev, t.ev[1:]):
            res.setdefault(b, []).append(ea.elapsed_time(eb))
print(" ".join(f"{k} {statistics.median(v):.4f}" for k, v in res.items()), "total",
      f"{sum(statistics.median(v) for v in res.values()):.4f} ms", sys.argv[1:])
