"""fp32 normalise of C5's curve set (616k moving-joint paths gathered from
the write pass rows), median of 7."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.curves import normalize_tensors  # noqa: E402
from paper_2208_14567_b200.solver import compact_valid, simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import native_batch  # noqa: E402

nb = native_batch(1_000_000, 5, 20, seed=5000)
topo, pos = torch.from_numpy(nb.topo).cuda(), torch.from_numpy(nb.pos).cuda()
res = simulate_tensors(pos, nb.table, 200, topo, write_traj=False, gate_only=True)
idx, cnt = compact_valid(res["first_t"], 200)
nv = int(cnt.item())
traj = torch.empty((nv * 20, 200, 2), dtype=torch.float32, device="cuda")
simulate_tensors(pos, nb.table, 200, topo, write_traj=True, traj=traj, traj_stride=20, cand=idx[:nv], coarse=False)
mv = torch.from_numpy(nb.types > 0).cuda()[topo[idx[:nv]].long()]
rows = (torch.arange(nv, device="cuda")[:, None] * 20 + torch.arange(20, device="cuda"))[mv]
ts = []
for i in range(9):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = normalize_tensors(traj, src_row=rows)
    e1.record()
    e1.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
print(f"normalise {rows.numel()} C5 curves: {statistics.median(ts):.3f} ms, unstable {int(r['unstable'].sum())}")
