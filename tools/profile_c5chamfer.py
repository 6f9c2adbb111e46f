"""C5 curve set + 64 queries, one multi-query chamfer scan (for ncu -k regex:chamfer_mq)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.atlas import chamfer_scan  # noqa: E402
from paper_2208_14567_b200.curves import normalize_tensors  # noqa: E402
from paper_2208_14567_b200.solver import compact_valid, simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import fourier_db, native_batch  # noqa: E402

nb = native_batch(1_000_000, 5, 20, seed=5000)
topo = torch.from_numpy(nb.topo).cuda()
pos = torch.from_numpy(nb.pos).cuda()
moving = torch.from_numpy(nb.types > 0).cuda()
res = simulate_tensors(pos, nb.table, 200, topo, write_traj=False, gate_only=True)
idx, cnt = compact_valid(res["first_t"], 200)
nv = int(cnt.item())
traj = torch.empty((nv * 20, 200, 2), dtype=torch.float32, device="cuda")
simulate_tensors(pos, nb.table, 200, topo, write_traj=True, traj=traj, traj_stride=20, cand=idx[:nv], coarse=False)
mv = moving[topo[idx[:nv]].long()]
rows = (torch.arange(nv, device="cuda")[:, None] * 20 + torch.arange(20, device="cuda"))[mv]
db = normalize_tensors(traj, src_row=rows)["out"]
queries = fourier_db(64, 200, seed=5151)
for _ in range(2):
    r = chamfer_scan(db, queries, k=10, threshold=0.0, mq_fine="fine" in sys.argv)
torch.cuda.synchronize()
print(r["n_stage"].tolist())
