"""Quick timing of the simulation kernels for A/B builds (one GPU):
C2 deferred pipeline (bench headline: screen, pending compaction, f64 path
writes, valid compaction) and a 1M-candidate 5-20 joint screen (C3 shape).

    python tools/time_sim.py [label]
"""
import hashlib
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.solver import PlanTable, simulate_deferred, simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import device_poses, mixed_batch, topology_pool  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else ""
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    for _ in range(3):
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


mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
pos = torch.from_numpy(mb.pos).cuda()
topo = torch.from_numpy(mb.topo).cuda()
table = mb.table()
traj = torch.empty((mb.B * 8, 200, 2), dtype=torch.float32, device="cuda")
res = {}


def c2():
    res["r"] = simulate_deferred(pos, table, 200, topo, traj=traj, dense_rows=True)


ms2 = timed(c2)
nv = int(res["r"]["valid_count"].item())
traj.zero_()  # digest run: rows never written stay zero
c2()
h = hashlib.sha256()
for k in ("first_t", "first_joint"):
    h.update(res["r"][k].cpu().numpy().tobytes())
h.update(traj[: int(res["r"]["pend_rows"].item())].cpu().numpy().tobytes())

mechs, plans = topology_pool(256, 5, 20, seed=3000)
t3 = PlanTable(plans)
B = 1_000_000
topo3 = (torch.arange(B, device="cuda") // 256 % len(plans)).to(torch.int32)
pos3 = device_poses(topo3, plans, 20, seed=77)


def c3():
    res["s"] = simulate_tensors(pos3, t3, 200, topo3, write_traj=False)


ms3 = timed(c3)
v3 = int((res["s"]["first_t"] == 200).sum().item())
for k in ("first_t", "first_joint"):
    h.update(res["s"][k].cpu().numpy().tobytes())
print(f"{label}: C2 deferred {ms2:.4f} ms ({1e5 / (ms2 / 1e3):.3e} sims/s, valid {nv}) | "
      f"C3-1M screen {ms3:.4f} ms ({B / (ms3 / 1e3):.3e} cand/s, valid {v3}), digest {h.hexdigest()[:16]}",
      flush=True)
