"""Print la_simulate's work counters for the C2 screen (fix-up replays etc.)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200 import _native as N  # noqa: E402
from paper_2208_14567_b200.solver import simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import mixed_batch  # noqa: E402

mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
pos = torch.from_numpy(mb.pos).cuda()
topo = torch.from_numpy(mb.topo).cuda()
table = mb.table()
names = ["fix lanes", "warp lane slots", "warp dyad slots", "cands", "replay rounds", "active lane-angles",
         "fp32 dyads", "reserved"]
for tau in (2e-4, 1e-4, 5e-5):
    for flags, label in ((N.LA_SIM_DEFER, "defer"), (0, "full")):
        ctr = torch.zeros(8, dtype=torch.int64, device="cuda")
        res = simulate_tensors(pos, table, 200, topo, write_traj=False, counters=ctr, fixup_tau=tau,
                               _extra_flags=flags)
        c = ctr.cpu().tolist()
        ft = res["first_t"]
        print(f"tau={tau} {label}: " + ", ".join(f"{n}={v}" for n, v in zip(names, c)),
              f"pending={int((ft == N.LA_PENDING).sum())} valid={int((ft == 200).sum())}", flush=True)
