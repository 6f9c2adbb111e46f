"""Diagnose fp32 screen flags / f64 trajectories vs the oracle per tau (GPU)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import links_oracle as O
from paper_2208_14567_b200.workloads import mixed_batch
from paper_2208_14567_b200.solver import PlanTable, simulate_tensors

for (lo, hi, cnt_c) in [(6, 8, 16384), (5, 20, 32768)]:
    mb = mixed_batch(cnt_c, lo, hi, seed=13, stride=20)
    dpos = torch.from_numpy(mb.pos).cuda(); dtopo = torch.from_numpy(mb.topo).cuda()
    refs = {}
    for t, p in enumerate(mb.plans):
        sel = np.flatnonzero(mb.topo == t)
        steps = [(s.target, s.a, s.b) for s in p.steps]
        refs[t] = (sel, O.simulate(mb.pos[sel][:, :p.n], steps, p.fixed, 200, with_margin=True))
    for tau in [0.0, 1e-6, 1e-5, 3e-5, 1e-4, 1e-3]:
        for write in (False, True):
            cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
            res = simulate_tensors(dpos, PlanTable(mb.plans), 200, topo=dtopo, traj_stride=20, fixup_tau=tau, counters=cnt, write_traj=write)
            ft = res["first_t"].cpu().numpy(); fj = res["first_joint"].cpu().numpy()
            bad = 0; near = 0; worst = 0.0
            for t, p in enumerate(mb.plans):
                sel, ref = refs[t]
                nr = ref["margin"] < 1e-6
                near += int(nr.sum())
                bad += int((((ft[sel] != ref["first_t"]) | (fj[sel] != ref["first_joint"])) & ~nr).sum())
                if write:
                    ok = np.flatnonzero((ref["first_t"] == 200) & (ft[sel] == 200))
                    if len(ok):
                        Pg = res["traj"].view(mb.B, 20, 200, 2)[torch.from_numpy(sel[ok]).cuda()][:, :p.n].cpu().numpy().astype(np.float64)
                        Pr = O.trajectories(ref)[ok]
                        err = np.abs(Pg - Pr).max(axis=(-1, -2))
                        lo_ = Pr.min(axis=-2); hi_ = Pr.max(axis=-2)
                        diag = np.hypot(hi_[..., 0] - lo_[..., 0], hi_[..., 1] - lo_[..., 1])
                        worst = max(worst, float((err / np.where(diag > 0, diag, 1)).max()))
            c = cnt.cpu().numpy()
            print(f"n={lo}..{hi} tau={tau:g} write={write}: flag mismatches {bad} (near-margin {near}), worst per-curve {worst:.2e}, fixups {c[0]}/{c[1]} = {c[0]/max(c[1],1):.4f}, dyads {c[2]}")
