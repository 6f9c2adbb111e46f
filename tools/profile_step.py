"""Small fixed workloads for ncu captures (one GPU).

    python tools/profile_step.py c2      # bench C2 pipeline: deferred screen, compaction, path writes
    python tools/profile_step.py c3      # screen of 1M candidates, 5-20 joints
    python tools/profile_step.py c4      # chamfer scan, 1 query x 1M curves
    python tools/profile_step.py norm    # normalise 200k fp32 paths
    python tools/profile_step.py filter  # coarse prefilter select over 10M descriptors
    python tools/profile_step.py gen     # generation (device poses, gate) + curve pipeline
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200 import _native  # noqa: E402

_native.load(build_if_missing=False)
what = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if what == "c2":
    from paper_2208_14567_b200.solver import simulate_deferred
    from paper_2208_14567_b200.workloads import mixed_batch

    mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
    pos = torch.from_numpy(mb.pos).cuda()
    topo = torch.from_numpy(mb.topo).cuda()
    table = mb.table()
    for _ in range(reps):
        simulate_deferred(pos, table, 200, topo, dense_rows=True)
elif what == "c3":
    from paper_2208_14567_b200.solver import PlanTable, simulate_tensors
    from paper_2208_14567_b200.workloads import device_poses, topology_pool

    mechs, plans = topology_pool(256, 5, 20, seed=3000)
    table = PlanTable(plans)
    B = 1_000_000
    topo = (torch.arange(B, device="cuda") // 256 % len(plans)).to(torch.int32)
    pos = device_poses(topo, plans, 20, seed=77)
    for _ in range(reps):
        simulate_tensors(pos, table, 200, topo, write_traj=False)
elif what == "c4":
    from paper_2208_14567_b200.atlas import chamfer_scan
    from paper_2208_14567_b200.workloads import fourier_db

    db = fourier_db(1_000_000, 200, seed=4000)
    q = fourier_db(1, 200, seed=999)
    for _ in range(reps):
        chamfer_scan(db, q, k=10)
elif what == "norm":
    from paper_2208_14567_b200.curves import normalize_tensors
    from paper_2208_14567_b200.workloads import fourier_curves_device

    raw = fourier_curves_device(200_000, 200, seed=5, dtype=torch.float32)
    for _ in range(reps):
        normalize_tensors(raw)
elif what == "c5":
    import bench as B

    class A:
        steps = 1
        warmup = 1

    class Clk:
        timed = False

    out = B.bench_c5(torch, A, 0, 1, {"sm_max_mhz": 1965.0, "hbm_gbs": 6551.7}, lambda: None, Clk)
    print({k: round(v, 3) for k, v in out["stages_ms"].items()})
elif what == "filter":
    from paper_2208_14567_b200.atlas import coarse_descriptors, coarse_select
    from paper_2208_14567_b200.workloads import fourier_curves_device

    raw = fourier_curves_device(1_000_000, 200, seed=6)
    desc = coarse_descriptors(raw)
    big = desc.repeat(10, 1)
    order = torch.randperm(big.shape[0], device="cuda")
    for _ in range(reps):
        coarse_select(big, desc[7], big.shape[0] // 100, order)
elif what == "gen":
    from paper_2208_14567_b200.dataset import curate_batch, curves_from_block
    from paper_2208_14567_b200.generator import GenerationConfig, GenerationRun

    for _ in range(reps):
        run = GenerationRun(GenerationConfig(count=5000, seed=1), traj_on_device=True, lookahead=8)
        for b in run.blocks():
            curate_batch(curves_from_block(b, 5), 0.005, 0)
torch.cuda.synchronize()
print("ok", what)
