"""C3 gate timing (bench workload: 10M 5-20 joint candidates, gate_only + low_t), median of 3."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.solver import simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import native_batch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
nb = native_batch(n, 5, 20, seed=3000)
pos, topo = torch.from_numpy(nb.pos).cuda(), torch.from_numpy(nb.topo).cuda()
ts = []
for i in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = simulate_tensors(pos, nb.table, 200, topo, write_traj=False, low=True, gate_only=True)
    e1.record()
    e1.synchronize()
    if i:
        ts.append(e0.elapsed_time(e1))
print(f"{sys.argv[2] if len(sys.argv) > 2 else ''} C3 {n}: {statistics.median(ts):.3f} ms, valid {int((r['first_t'] == 200).sum())}")
