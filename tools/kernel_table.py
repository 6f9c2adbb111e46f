"""Launch every kernel of the library once at a representative size (for an
ncu metrics pass that tabulates achieved HBM GB/s and FP32 FLOP/s per kernel:
tools/ncu_table.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_14567_b200 import _native as N  # noqa: E402

N.load(build_if_missing=False)
from paper_2208_14567_b200.atlas import chamfer_scan, coarse_descriptors, coarse_select  # noqa: E402
from paper_2208_14567_b200.curves import circle_stats, normalize_tensors  # noqa: E402
from paper_2208_14567_b200.dataset import curation_keep_batch  # noqa: E402
from paper_2208_14567_b200.generator import GenerationConfig, GenerationRun  # noqa: E402
from paper_2208_14567_b200.solver import dyad_solve, plan_geometry, simulate_deferred, simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import fourier_curves_device, fourier_db, four_bar, bare_plan, mixed_batch  # noqa: E402

mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
pos = torch.from_numpy(mb.pos).cuda()
topo = torch.from_numpy(mb.topo).cuda()
table = mb.table()
res = simulate_deferred(pos, table, 200, topo)                         # screen, compaction x2, write-only
simulate_deferred(pos, table, 200, topo, split_rows=True)              # split-row compaction + split write
simulate_tensors(pos, table, 200, topo, write_traj=False, _extra_flags=N.LA_SIM_LANE_SCREEN)  # lane screen
from paper_2208_14567_b200.workloads import native_batch  # noqa: E402
nb = native_batch(200_000, 5, 20, seed=3000)
simulate_tensors(torch.from_numpy(nb.pos).cuda(), nb.table, 200, torch.from_numpy(nb.topo).cuda(),
                 write_traj=False, gate_only=True, low=True)           # 20-joint screen (fp16 error slots)
simulate_tensors(pos, table, 200, topo, write_traj=True, traj_f64=True, traj_stride=8)  # exact f64 writes
mech = four_bar()
plan = bare_plan(mech)
plan_geometry(plan, mech.positions0)                                   # geometry_kernel
dyad_solve(np.array([0.5, 0.5]), np.array([0.7, 0.5]), 0.15, 0.12, 1.0)  # dyad_kernel
raw = fourier_curves_device(200_000, 200, seed=5, dtype=torch.float32)
normalize_tensors(raw)                                                 # normalize_warp_kernel (fp32)
raw64 = fourier_curves_device(20_000, 200, seed=6)
n64 = normalize_tensors(raw64, out_f64=True)                           # normalize_kernel<double>
circle_stats(n64["out"])                                               # circle_kernel
db = fourier_db(1_000_000, 200, seed=4000)
q = fourier_db(64, 200, seed=999)
chamfer_scan(db, q[:1], k=10)                                          # chamfer scan + select/merge
from paper_2208_14567_b200.atlas import chamfer_index  # noqa: E402
chamfer_scan(db, q[:1], k=10, cells=chamfer_index(db))                 # cell index, bound step, survivors' scan
chamfer_scan(db[:200_000], q, k=10)                                    # 64 queries: multi-query kernel
chamfer_scan(db[:200_000], q, k=10, multi_query=False)                 # 64 queries, one CTA set each
from paper_2208_14567_b200.dist import merge_gathered, pack_lists  # noqa: E402
parts = [chamfer_scan(db[i * 100_000:(i + 1) * 100_000], q[:8], k=10, id_base=i * 100_000,
                      pos_base=i * 100_000) for i in range(2)]
merge_gathered(torch.stack([pack_lists(p_, 10) for p_ in parts]), 10)  # shard_merge_kernel
desc = coarse_descriptors(raw64)                                       # descriptor_kernel
big = desc.repeat(50, 1)
coarse_select(big, desc[3], big.shape[0] // 100, torch.randperm(big.shape[0], device="cuda"))
ids = np.arange(1_000_000)
curation_keep_batch(ids, ids % 20, np.ones(len(ids), bool), 0.005, 3)  # curation_keep_kernel
run = GenerationRun(GenerationConfig(count=5000, seed=1), traj_on_device=True, lookahead=8)
for b in run.blocks():
    pass                                                               # gen_poses_kernel + gate
torch.cuda.synchronize()
print("ok")
