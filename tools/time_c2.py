import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2208_14567_b200.solver import simulate_tensors, compact_valid
from paper_2208_14567_b200.workloads import mixed_batch
mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
pos = torch.from_numpy(mb.pos).cuda(); topo = torch.from_numpy(mb.topo).cuda(); table = mb.table()
traj = torch.empty((mb.B * 8, 200, 2), dtype=torch.float32, device="cuda")
for it in range(6):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    h = []
    torch.cuda.synchronize()
    t0 = time.perf_counter(); ev[0].record()
    r = simulate_tensors(pos, table, 200, topo, write_traj=False); h.append(time.perf_counter() - t0); ev[1].record()
    idx, cnt = compact_valid(r["first_t"], 200); h.append(time.perf_counter() - t0); ev[2].record()
    simulate_tensors(pos, table, 200, topo, write_traj=True, traj=traj, traj_stride=8, cand=idx, cand_count=cnt, coarse=False); h.append(time.perf_counter() - t0); ev[3].record()
    torch.cuda.synchronize(); h.append(time.perf_counter() - t0)
    print("gpu ms", [round(ev[i].elapsed_time(ev[i+1]), 4) for i in range(3)], "host ms", [round(x*1e3, 3) for x in h])
