"""One C2 deferred screen (lane kernel unless 'warp' given) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200 import _native as N  # noqa: E402
from paper_2208_14567_b200.solver import simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import mixed_batch, native_batch  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
extra = 0 if "warp" in sys.argv else N.LA_SIM_LANE_SCREEN
if which == "c2":
    mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
    pos, table, topo = torch.from_numpy(mb.pos).cuda(), mb.table(), torch.from_numpy(mb.topo).cuda()
    kw = dict(_extra_flags=extra | N.LA_SIM_DEFER)
else:
    nb = native_batch(500_000, 5, 20, seed=3000)
    pos, table, topo = torch.from_numpy(nb.pos).cuda(), nb.table, torch.from_numpy(nb.topo).cuda()
    kw = dict(_extra_flags=extra, gate_only=True, low=True)
for _ in range(3):
    simulate_tensors(pos, table, 200, topo, write_traj=False, **kw)
torch.cuda.synchronize()
