"""Flag mismatches of the fp32 screen (with f64 fix-up below tau) against
the all-f64 exact mode, per tau, on C2 and on 5-20 joint candidates."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.solver import simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import mixed_batch, native_batch  # noqa: E402

sets = []
mb = mixed_batch(100_000, 6, 8, seed=2208, stride=8)
sets.append(("C2 6-8", torch.from_numpy(mb.pos).cuda(), torch.from_numpy(mb.topo).cuda(), mb.table()))
for seed in (1, 2):
    nb = native_batch(2_000_000, 5, 20, seed=900 + seed)
    sets.append((f"5-20 #{seed}", torch.from_numpy(nb.pos).cuda(), torch.from_numpy(nb.topo).cuda(), nb.table))
for name, pos, topo, table in sets:
    ref = simulate_tensors(pos, table, 200, topo, write_traj=False, fp64=True, exact=True)
    for tau in [float(x) for x in os.environ.get("TAUS", "2e-4,1e-4,5e-5,2e-5,1e-5,5e-6,0").split(",")]:
        ctr = torch.zeros(8, dtype=torch.int64, device="cuda")
        res = simulate_tensors(pos, table, 200, topo, write_traj=False, fixup_tau=tau, counters=ctr)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        simulate_tensors(pos, table, 200, topo, write_traj=False, fixup_tau=tau)
        e1.record()
        e1.synchronize()
        bad = int(((res["first_t"] != ref["first_t"]) | (res["first_joint"] != ref["first_joint"])).sum())
        c = ctr.cpu().tolist()
        print(f"{name}: B={pos.shape[0]} tau={tau:g}: {bad} flag mismatches vs exact f64; fix lanes {c[0]}, "
              f"replay rounds {c[4]}, {e0.elapsed_time(e1):.3f} ms", flush=True)
