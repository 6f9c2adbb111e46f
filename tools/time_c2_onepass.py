"""C2: deferred pipeline (screen -> compaction -> f64 write pass) vs the
one-pass write mode (each warp screens its candidate and writes its paths at
once, sparse rows i * stride), both timed with CUDA events after an L2
flush; median of 10."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.solver import DeferredGraph, compact_valid, simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import mixed_batch  # noqa: E402

mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
pos, topo, table = torch.from_numpy(mb.pos).cuda(), torch.from_numpy(mb.topo).cuda(), mb.table()
traj = torch.empty((mb.B * 8, 200, 2), dtype=torch.float32, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


g = DeferredGraph(pos, table, 200, topo, traj=traj)
print(f"deferred graph  {timed(g.replay):.4f} ms", flush=True)


def onepass():
    r = simulate_tensors(pos, table, 200, topo, write_traj=True, traj=traj, traj_stride=8)
    compact_valid(r["first_t"], 200)


print(f"one-pass write  {timed(onepass):.4f} ms", flush=True)
r = simulate_tensors(pos, table, 200, topo, write_traj=True, traj=traj, traj_stride=8)
print("flags equal:", bool(torch.equal(r["first_t"], g.out["first_t"])), flush=True)
