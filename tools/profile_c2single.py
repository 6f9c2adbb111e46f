import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2208_14567_b200.solver import simulate_tensors
from paper_2208_14567_b200.workloads import mixed_batch
mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
pos = torch.from_numpy(mb.pos).cuda(); topo = torch.from_numpy(mb.topo).cuda(); table = mb.table()
traj = torch.empty((mb.B * 8, 200, 2), dtype=torch.float32, device="cuda")
for _ in range(3):
    simulate_tensors(pos, table, 200, topo, write_traj=True, traj=traj, traj_stride=8)
torch.cuda.synchronize()
print("ok")
