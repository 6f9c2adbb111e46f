"""GPU parity of the simulation / screening kernel against the reference
(golden fixtures) and the oracle (seeded subsets).  Tolerances follow
BASELINE.json north_star / SURVEY.md §8a:

* lock flags (first_t, first_joint) bit-exact except candidates whose f64
  discriminant margin is below 1e-6 (counted, reported);
* fp32 coordinates within 1e-4 of the reference path's bounding-box
  diagonal, floored at 1e-3 of the unit box (below that an fp32-stored
  coordinate near 0.5 cannot resolve 1e-4 of the diagonal: half an ulp is
  3e-8); f64 trajectories (the drop-in API) within 1e-12 absolute.
"""

import numpy as np
import pytest

from oracle import links_oracle as O

pytestmark = pytest.mark.gpu

MARGIN = 1e-6
COORD_TOL = 1e-4
DIAG_FLOOR = 1e-3
F64_TOL = 1e-12


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def bbox_diag(P):
    lo = np.nanmin(P, axis=-2)
    hi = np.nanmax(P, axis=-2)
    return np.hypot(*(hi - lo).T) if P.ndim == 2 else np.hypot(hi[..., 0] - lo[..., 0], hi[..., 1] - lo[..., 1])


def coord_err(P_gpu, P_ref):
    """max over joint paths of max |dP| / max(bbox diagonal, DIAG_FLOOR)."""
    err = np.abs(P_gpu - P_ref).max(axis=(-1, -2))  # (..., n)
    diag = np.maximum(bbox_diag(P_ref), DIAG_FLOOR)
    return float((err / diag).max())


def flag_parity(ft, fj, ref_ft, ref_fj, margin):
    near = margin < MARGIN
    bad = ((ft != ref_ft) | (fj != ref_fj)) & ~near
    return int(bad.sum()), int(near.sum())


def run_mixed(torch, plans, pos, topo, T, **kw):
    from paper_2208_14567_b200.solver import PlanTable, simulate_tensors

    dpos = torch.from_numpy(np.ascontiguousarray(pos)).cuda()
    dtopo = None if topo is None else torch.from_numpy(np.ascontiguousarray(topo, dtype=np.int32)).cuda()
    res = simulate_tensors(dpos, PlanTable(plans), T, topo=dtopo, traj_stride=pos.shape[1], **kw)
    torch.cuda.synchronize()
    return res


def test_fourbar_golden(torch, golden):
    from paper_2208_14567_b200.workloads import bare_plan, four_bar

    g = golden("solver_golden.npz")
    plan = bare_plan(four_bar())
    res = run_mixed(torch, [plan], g["fb_pos0"], None, 200, low=True)
    ft = res["first_t"].cpu().numpy()
    fj = res["first_joint"].cpu().numpy()
    margin = O.simulate(g["fb_pos0"], [(3, 1, 2)], (0, 2), 200, with_margin=True)["margin"]
    bad, near = flag_parity(ft, fj, g["fb_first_t"], g["fb_first_joint"], margin)
    assert bad == 0, f"{bad} flag mismatches outside the margin band ({near} near-margin)"
    # the coarse sweep is the T_low = 50 gate of the reference
    low = res["low_t"].cpu().numpy()
    want_low = np.where(g["fb_first_t50"] < 50, g["fb_first_t50"], -1)
    assert np.array_equal(low[margin >= MARGIN], want_low[margin >= MARGIN])
    traj = res["traj"].view(-1, 4, 200, 2).cpu().numpy().astype(np.float64)
    assert coord_err(traj[g["fb_traj_idx"]], g["fb_traj"]) <= COORD_TOL
    r64 = run_mixed(torch, [plan], g["fb_pos0"], None, 200, traj_f64=True)
    t64 = r64["traj"].view(-1, 4, 200, 2).cpu().numpy()
    assert np.abs(t64[g["fb_traj_idx"]] - g["fb_traj"]).max() <= F64_TOL
    assert torch.equal(r64["first_t"], res["first_t"])


def test_mixed_topologies_golden(torch, golden):
    from paper_2208_14567_b200.solver import SolutionPlan, compile_order

    g = golden("solver_golden.npz")
    plans = []
    for t in range(len(g["mx_n"])):
        n = int(g["mx_n"][t])
        fixed, steps = compile_order(g["mx_adj"][t][:n, :n], g["mx_types"][t][:n])
        plans.append(SolutionPlan(n, fixed, steps, None, None, None))
    pos = g["mx_pos0"]
    res = run_mixed(torch, plans, pos, g["mx_topo"], 200, low=True)
    ft = res["first_t"].cpu().numpy()
    fj = res["first_joint"].cpu().numpy()
    margins = np.empty(len(ft))
    for t, p in enumerate(plans):
        sel = g["mx_topo"] == t
        steps = [(s.target, s.a, s.b) for s in p.steps]
        margins[sel] = O.simulate(pos[sel][:, :p.n], steps, p.fixed, 200, with_margin=True)["margin"]
    bad, near = flag_parity(ft, fj, g["mx_first_t"], g["mx_first_joint"], margins)
    assert bad == 0, f"{bad} mismatches ({near} near-margin)"
    traj = res["traj"].view(len(ft), 20, 200, 2).cpu().numpy().astype(np.float64)
    for gi, tp in zip(g["mx_traj_idx"], g["mx_traj"]):
        n = int(g["mx_n"][g["mx_topo"][gi]])
        assert ft[gi] == 200
        assert coord_err(traj[gi, :n], tp[:n]) <= COORD_TOL


def test_screen_mode_matches_simulate_mode(torch, golden):
    """No-write screening (coarse-first, fine search) == full simulation."""
    from paper_2208_14567_b200.solver import SolutionPlan, compile_order

    g = golden("solver_golden.npz")
    plans = []
    for t in range(len(g["mx_n"])):
        n = int(g["mx_n"][t])
        fixed, steps = compile_order(g["mx_adj"][t][:n, :n], g["mx_types"][t][:n])
        plans.append(SolutionPlan(n, fixed, steps, None, None, None))
    a = run_mixed(torch, plans, g["mx_pos0"], g["mx_topo"], 200)
    b = run_mixed(torch, plans, g["mx_pos0"], g["mx_topo"], 200, write_traj=False)
    c = run_mixed(torch, plans, g["mx_pos0"], g["mx_topo"], 200, write_traj=False, coarse=False)
    for k in ("first_t", "first_joint"):
        assert torch.equal(a[k], b[k]) and torch.equal(a[k], c[k])


def test_fp64_mode_and_no_fixup(torch, golden):
    """All-f64 evaluation agrees with the reference flags; tau=0 (pure fp32)
    still matches outside the margin band on this fixture."""
    from paper_2208_14567_b200.workloads import bare_plan, four_bar

    g = golden("solver_golden.npz")
    plan = bare_plan(four_bar())
    margin = O.simulate(g["fb_pos0"], [(3, 1, 2)], (0, 2), 200, with_margin=True)["margin"]
    for kw in ({"fp64": True}, {"fixup_tau": 0.0}):
        res = run_mixed(torch, [plan], g["fb_pos0"], None, 200, **kw)
        bad, _ = flag_parity(res["first_t"].cpu().numpy(), res["first_joint"].cpu().numpy(),
                             g["fb_first_t"], g["fb_first_joint"], margin)
        assert bad == 0, kw
    res = run_mixed(torch, [plan], g["fb_pos0"], None, 200, fp64=True, traj_f64=True)
    traj = res["traj"].view(-1, 4, 200, 2).cpu().numpy()
    assert np.abs(traj[g["fb_traj_idx"]] - g["fb_traj"]).max() <= F64_TOL


def test_known_answers(torch, golden):
    from paper_2208_14567_b200 import Locking, Trajectory, compile_plan, dyad_solve, simulate
    from paper_2208_14567_b200.workloads import four_bar

    g = golden("solver_golden.npz")
    p = dyad_solve((0.0, 0.0), (1.0, 0.0), 1.0, 1.0, 1.0)
    assert p == (0.5, 0.8660254037844386)
    q = dyad_solve((0.0, 0.0), (2.0, 0.0), 1.5, 1.5, -1.0)
    assert q[0] == pytest.approx(1.0) and q[1] < 0
    assert dyad_solve((0.0, 0.0), (2.0, 0.0), 0.5, 0.5, 1.0) is None
    assert dyad_solve((0.0, 0.0), (0.0, 0.0), 1.0, 1.0, 1.0) is None
    lock = four_bar(ground=(0.9, 0.5), coupler=(0.72, 0.51))
    plan = compile_plan(lock)
    o200 = simulate(lock, plan, 200)
    o50 = simulate(lock, plan, 50)
    assert isinstance(o200, Locking) and (o200.step, o200.joint) == tuple(g["ka_lock"][:2])
    assert isinstance(o50, Locking) and o50.step == g["ka_lock"][2]
    ok = four_bar()
    out = simulate(ok, compile_plan(ok), 200)
    assert isinstance(out, Trajectory)
    assert np.abs(out.positions - g["ka_valid_traj"]).max() <= F64_TOL
    assert np.allclose(out.positions[:, 0, :], ok.positions0, atol=1e-12)


def test_plan_geometry_and_compile_plan(torch):
    from paper_2208_14567_b200 import PlanError, compile_plan
    from paper_2208_14567_b200.solver import plan_geometry
    from paper_2208_14567_b200.workloads import four_bar

    m = four_bar()
    plan = compile_plan(m)
    ra, rb, br = plan_geometry(plan, m.positions0)
    wa, wb, wbr = O.step_geometry(m.positions0[None], [(3, 1, 2)])
    assert np.allclose(ra, wa[0], rtol=0, atol=1e-15) and np.allclose(rb, wb[0], rtol=0, atol=1e-15)
    assert np.array_equal(br, wbr[0])
    assert plan.fixed == (0, 2) and [s.target for s in plan.steps] == [3]
    degenerate = four_bar(coupler=(0.55, 0.5))  # joint 3 on the crank tip: zero bar
    with pytest.raises(PlanError):
        compile_plan(degenerate)


def test_simulate_batch_dropin_conserves_lengths(torch):
    from paper_2208_14567_b200 import Trajectory, compile_plan, simulate_batch
    from paper_2208_14567_b200.workloads import four_bar

    rng = np.random.default_rng(5)
    mech = four_bar()
    plan = compile_plan(mech)
    poses = []
    for _ in range(64):
        p = np.array(mech.positions0)
        p[2] = rng.uniform(0.2, 0.9, size=2)
        p[3] = rng.uniform(0.2, 0.9, size=2)
        poses.append(p)
    poses = np.stack(poses)
    outs = simulate_batch(poses, plan, T=100)
    ref = O.simulate(poses, [(3, 1, 2)], (0, 2), 100, with_margin=True)
    for b, o in enumerate(outs):
        if ref["margin"][b] < MARGIN:
            continue
        if ref["first_t"][b] < 100:
            assert not isinstance(o, Trajectory) and o.step == ref["first_t"][b]
        else:
            assert isinstance(o, Trajectory)
            P = o.positions
            assert np.abs(P - O.trajectories(ref)[b]).max() <= F64_TOL
            for i, j in mech.edges():
                L = np.hypot(*(P[i] - P[j]).T)
                assert L.max() - L.min() < 1e-9  # the reference's own bound


def test_check_feasible_and_find_valid_variant(torch, golden):
    from paper_2208_14567_b200 import check_feasible, find_valid_variant, sample_topology
    from paper_2208_14567_b200.solver import SolutionPlan, compile_order

    g = golden("solver_golden.npz")
    for t in range(len(g["fv_n"])):
        n = int(g["fv_n"][t])
        seed = int(g["fv_seed"][t])
        mech, plan = sample_topology(np.random.default_rng([seed, 0]), n)
        rng = np.random.default_rng([seed, 1])
        res = find_valid_variant(mech, plan, rng)
        assert res is not None
        assert res.attempts == int(g["fv_attempts"][t])
        assert np.array_equal(res.mechanism.positions0, g["fv_pos"][t][:n])
        assert check_feasible(res.mechanism, plan)
        # rng left exactly where the reference loop leaves it
        ref_rng = np.random.default_rng([seed, 1])
        batches = (int(g["fv_attempts"][t]) + 255) // 256
        for _ in range(batches):
            ref_rng.uniform(size=(256, n, 2))
        assert rng.random() == ref_rng.random()
    # non-fused path (T_high != 4*T_low) agrees on the same stream
    n = int(g["fv_n"][0])
    seed = int(g["fv_seed"][0])
    mech, plan = sample_topology(np.random.default_rng([seed, 0]), n)
    a = find_valid_variant(mech, plan, np.random.default_rng([seed, 1]), T_low=40, T_high=200)
    assert a is not None and a.attempts >= 1


@pytest.mark.parametrize("n_lo,n_hi,count", [(6, 8, 8192), (5, 20, 16384)])
def test_mixed_scale_vs_oracle(torch, n_lo, n_hi, count):
    """C2 / C3-style candidates from the generator streams: flags vs the
    oracle with the margin rule; coordinates within 1e-4 of the diagonal."""
    from paper_2208_14567_b200.workloads import mixed_batch

    mb = mixed_batch(count, n_lo, n_hi, seed=11, stride=20)
    res = run_mixed(torch, mb.plans, mb.pos, mb.topo, 200, low=True)
    ft = res["first_t"].cpu().numpy()
    fj = res["first_joint"].cpu().numpy()
    traj = res["traj"].view(mb.B, 20, 200, 2)
    total_bad = total_near = 0
    worst = 0.0
    tiny = 0
    for t, p in enumerate(mb.plans):
        sel = np.flatnonzero(mb.topo == t)
        steps = [(s.target, s.a, s.b) for s in p.steps]
        ref = O.simulate(mb.pos[sel][:, :p.n], steps, p.fixed, 200, with_margin=True)
        bad, near = flag_parity(ft[sel], fj[sel], ref["first_t"], ref["first_joint"], ref["margin"])
        total_bad += bad
        total_near += near
        ok = np.flatnonzero((ref["first_t"] == 200) & (ft[sel] == 200))
        if len(ok):
            Pg = traj[torch.from_numpy(sel[ok]).cuda()][:, :p.n].cpu().numpy().astype(np.float64)
            Pr = O.trajectories(ref)[ok]
            worst = max(worst, coord_err(Pg, Pr))
            tiny += int((bbox_diag(Pr) < DIAG_FLOOR).sum())
    print(f"\nmixed n={n_lo}..{n_hi}: {count} candidates, valid {(ft == 200).mean():.3f}, "
          f"near-margin {total_near}, flag mismatches {total_bad}, worst coord err {worst:.2e}, "
          f"paths with diagonal < {DIAG_FLOOR}: {tiny}")
    assert total_bad == 0
    assert worst <= COORD_TOL


def test_compaction_ordered(torch):
    from paper_2208_14567_b200.solver import compact_valid

    gen = torch.Generator(device="cuda").manual_seed(3)
    for B in (1, 1000, 1024, 1025, 300_001):
        ft = torch.randint(150, 201, (B,), generator=gen, device="cuda", dtype=torch.int32)
        idx, cnt = compact_valid(ft, 200)
        want = torch.nonzero(ft == 200).flatten()
        assert int(cnt.item()) == want.numel()
        assert torch.equal(idx[: want.numel()], want)


def test_compaction_lookback_edges(torch):
    """The single-pass look-back selection: none / all selected, sizes around
    a tile, a few thousand tiles (look-back over many published aggregates),
    and the split row sums of la_compact_rows_split against numpy."""
    from paper_2208_14567_b200.solver import compact_rows_split, compact_valid
    from paper_2208_14567_b200.workloads import mixed_batch

    for B, fill in ((5000, 0), (5000, 200), (2_500_003, None)):
        ft = (torch.full((B,), fill, dtype=torch.int32, device="cuda") if fill is not None else
              torch.randint(190, 201, (B,), device="cuda", dtype=torch.int32))
        idx, cnt = compact_valid(ft, 200)
        want = torch.nonzero(ft == 200).flatten()
        assert int(cnt.item()) == want.numel()
        assert torch.equal(idx[: want.numel()], want)
    mb = mixed_batch(70_000, 5, 12, seed=29, stride=12)
    table = mb.table()
    topo = torch.from_numpy(mb.topo).cuda()
    ft = torch.randint(198, 201, (mb.B,), device="cuda", dtype=torch.int32)
    idx, row, row2, cnt, tot, tot2 = compact_rows_split(ft, 200, table, topo)
    sel = np.flatnonzero(ft.cpu().numpy() == 200)
    ns = np.array([len(p.steps) for p in mb.plans])[mb.topo[sel]]
    n = mb.n[sel]
    k = int(cnt.item())
    assert k == len(sel) and np.array_equal(idx[:k].cpu().numpy(), sel)
    assert np.array_equal(row[:k].cpu().numpy(), np.concatenate([[0], np.cumsum(ns)[:-1]]))
    assert np.array_equal(row2[:k].cpu().numpy(), np.concatenate([[0], np.cumsum(n - ns)[:-1]]))
    assert int(tot.item()) == int(ns.sum()) and int(tot2.item()) == int((n - ns).sum())


def test_gate_only_flag(torch, golden):
    """LA_SIM_GATE_ONLY: negatives carry the coarse lock, positives exact."""
    from paper_2208_14567_b200.workloads import bare_plan, four_bar

    g = golden("solver_golden.npz")
    res = run_mixed(torch, [bare_plan(four_bar())], g["fb_pos0"], None, 200, write_traj=False,
                    gate_only=True, low=True)
    ft = res["first_t"].cpu().numpy()
    low = res["low_t"].cpu().numpy()
    assert np.array_equal(ft == 200, g["fb_first_t"] == 200)
    locked = low >= 0
    assert np.array_equal(ft[locked], 4 * low[locked])


def test_cand_gather_and_device_count(torch, golden):
    """Work-item gathering: cand subset (no count) and cand + device count
    give the full-batch results at the gathered indices."""
    from paper_2208_14567_b200.solver import PlanTable, SolutionPlan, compile_order, simulate_tensors

    g = golden("solver_golden.npz")
    plans = []
    for t in range(len(g["mx_n"])):
        n = int(g["mx_n"][t])
        fixed, steps = compile_order(g["mx_adj"][t][:n, :n], g["mx_types"][t][:n])
        plans.append(SolutionPlan(n, fixed, steps, None, None, None))
    full = run_mixed(torch, plans, g["mx_pos0"], g["mx_topo"], 200)
    sel = torch.from_numpy(np.random.default_rng(1).choice(len(g["mx_topo"]), 300, replace=False)).cuda()
    pos = torch.from_numpy(g["mx_pos0"]).cuda()
    topo = torch.from_numpy(g["mx_topo"]).cuda()
    part = simulate_tensors(pos, PlanTable(plans), 200, topo, traj_stride=20, cand=sel)
    assert torch.equal(part["first_t"], full["first_t"][sel])
    ok = (part["first_t"] == 200).nonzero().flatten()
    a = part["traj"].view(300, 20, 200, 2)[ok]
    b = full["traj"].view(-1, 20, 200, 2)[sel[ok]]
    for i in range(len(ok)):
        n = plans[int(g["mx_topo"][int(sel[ok[i]])])].n
        assert torch.equal(a[i, :n], b[i, :n])
    cnt = torch.tensor([100], dtype=torch.int64, device="cuda")
    part2 = simulate_tensors(pos, PlanTable(plans), 200, topo, write_traj=False, cand=sel, cand_count=cnt)
    torch.cuda.synchronize()
    assert torch.equal(part2["first_t"][:100], full["first_t"][sel[:100]])


@pytest.mark.parametrize("T", [1, 2, 8, 50, 100, 199, 201, 360, 2048])
def test_other_T_values(torch, golden, T):
    """Coarse-first order needs T % 4 == 0; other T take the plain order.
    Flags and f64 paths match the oracle for any T."""
    from paper_2208_14567_b200.solver import SolutionPlan, compile_order

    g = golden("solver_golden.npz")
    t = 25  # an n = 18 topology of the fixture
    n = int(g["mx_n"][t])
    fixed, steps = compile_order(g["mx_adj"][t][:n, :n], g["mx_types"][t][:n])
    plan = SolutionPlan(n, fixed, steps, None, None, None)
    fb = [(s.target, s.a, s.b) for s in steps]
    pos = g["mx_pos0"][g["mx_topo"] == t][:, :n]
    # plus the four-bar batch (mostly valid) to exercise the path writes
    from paper_2208_14567_b200.workloads import bare_plan, four_bar

    for plan_, fb_, fixed_, P in ((plan, fb, fixed, pos), (bare_plan(four_bar()), [(3, 1, 2)], (0, 2),
                                                           g["fb_pos0"][:64])):
        ref = O.simulate(P, fb_, fixed_, T, with_margin=True)
        res = run_mixed(torch, [plan_], P, None, T, traj_f64=True)
        bad, _ = flag_parity(res["first_t"].cpu().numpy(), res["first_joint"].cpu().numpy(), ref["first_t"],
                             ref["first_joint"], ref["margin"])
        assert bad == 0
        ok = np.flatnonzero((ref["first_t"] == T) & (res["first_t"].cpu().numpy() == T))
        tr = res["traj"].view(len(P), plan_.n, T, 2).cpu().numpy()
        if len(ok):  # exact f64 mode: bit-identical to the reference order of operations
            assert np.array_equal(tr[ok], O.trajectories(ref)[ok])


def test_edge_cases(torch):
    from paper_2208_14567_b200 import simulate_batch
    from paper_2208_14567_b200._native import NativeError
    from paper_2208_14567_b200.solver import PlanTable, SolutionPlan, simulate_tensors
    from paper_2208_14567_b200.workloads import bare_plan, four_bar

    plan = bare_plan(four_bar())
    assert simulate_batch(np.zeros((0, 4, 2)), plan) == []
    # a plan with more joints than the pose stride is flagged, not read out of bounds
    big = SolutionPlan(6, (0, 2), plan.steps, None, None, None)
    pos = torch.rand((3, 4, 2), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        simulate_tensors(pos, PlanTable([big]), 200)
    with pytest.raises(NativeError):
        simulate_tensors(pos, PlanTable([plan]), 4096)  # T beyond the compiled limit
    # coincident joints lock (d < LOCK_EPS), like the reference
    p = np.array(four_bar().positions0)[None].repeat(2, 0)
    p[1, 2] = p[1, 1]  # ground joint on the crank tip at t = 0: d(1, 2) = 0 at t = 0
    ref = O.simulate(p, [(3, 1, 2)], (0, 2), 200)
    outs = simulate_batch(p, plan, 200)
    for o, ft in zip(outs, ref["first_t"]):
        assert (getattr(o, "step", 200)) == ft


def test_deferred_pipeline_matches_single_pass(torch):
    """screen(defer) -> compact -> f64 write-only scatter == single pass."""
    from paper_2208_14567_b200.solver import simulate_deferred
    from paper_2208_14567_b200.workloads import mixed_batch

    mb = mixed_batch(6000, 5, 20, seed=21, stride=20)
    pos = torch.from_numpy(mb.pos).cuda()
    topo = torch.from_numpy(mb.topo).cuda()
    ref = run_mixed(torch, mb.plans, mb.pos, mb.topo, 200)
    res = simulate_deferred(pos, mb.table(), 200, topo)
    torch.cuda.synchronize()
    assert torch.equal(res["first_t"], ref["first_t"])
    assert torch.equal(res["first_joint"], ref["first_joint"])
    np_ = int(res["pend_count"].item())
    pend = res["pend_idx"][:np_]
    assert bool((ref["first_t"][pend] > 0).all())
    ok = (res["first_t"][pend] == 200).nonzero().flatten()
    a = res["traj"].view(-1, 20, 200, 2)[ok]
    b = ref["traj"].view(-1, 20, 200, 2)[pend[ok]]
    for i in range(len(ok)):
        n = int(mb.n[int(pend[ok[i]])])
        assert torch.equal(a[i, :n], b[i, :n])
    nv = int(res["valid_count"].item())
    assert torch.equal(res["valid_idx"][:nv], (ref["first_t"] == 200).nonzero().flatten())


def test_deferred_dense_rows(torch):
    """dense_rows (la_compact_rows): the same pending list, row offsets are
    the running sum of the pending candidates' joint counts, and each
    candidate's rows equal its strided rows bit for bit (no padding rows)."""
    from paper_2208_14567_b200.solver import simulate_deferred
    from paper_2208_14567_b200.workloads import mixed_batch

    mb = mixed_batch(6000, 5, 20, seed=22, stride=20)
    pos = torch.from_numpy(mb.pos).cuda()
    topo = torch.from_numpy(mb.topo).cuda()
    a = simulate_deferred(pos, mb.table(), 200, topo)
    d = simulate_deferred(pos, mb.table(), 200, topo, dense_rows=True)
    torch.cuda.synchronize()
    assert torch.equal(a["first_t"], d["first_t"]) and torch.equal(a["first_joint"], d["first_joint"])
    npend = int(a["pend_count"].item())
    assert int(d["pend_count"].item()) == npend
    pend = a["pend_idx"][:npend].cpu().numpy()
    assert np.array_equal(d["pend_idx"][:npend].cpu().numpy(), pend)
    n = mb.n[pend].astype(np.int64)
    off = np.concatenate([[0], np.cumsum(n)[:-1]])
    assert np.array_equal(d["pend_row"][:npend].cpu().numpy(), off)
    assert int(d["pend_rows"].item()) == int(n.sum())
    ta = a["traj"].view(-1, 20, 200, 2).cpu()
    td = d["traj"].cpu()
    ft = d["first_t"].cpu().numpy()
    for i in range(npend):
        if ft[pend[i]] == 200:
            assert torch.equal(td[off[i]:off[i] + n[i]], ta[i, :n[i]])
    # nothing selected / everything selected
    from paper_2208_14567_b200.solver import compact_rows

    ft0 = torch.zeros(3000, dtype=torch.int32, device="cuda")
    _, _, c0, r0 = compact_rows(ft0, 7, mb.table(), topo[:3000])
    assert int(c0.item()) == 0 and int(r0.item()) == 0
    idx, row, c1, r1 = compact_rows(ft0, 0, mb.table(), topo[:3000])
    nn = mb.n[:3000].astype(np.int64)
    assert int(c1.item()) == 3000 and int(r1.item()) == int(nn.sum())
    assert np.array_equal(idx[:3000].cpu().numpy(), np.arange(3000))
    assert np.array_equal(row[:3000].cpu().numpy(), np.concatenate([[0], np.cumsum(nn)[:-1]]))


def test_deferred_graph_replay(torch):
    """DeferredGraph (the deferred pipeline captured as CUDA graphs) equals
    simulate_deferred, and a replay after new poses are copied into its
    input buffer recomputes everything."""
    from paper_2208_14567_b200.solver import DeferredGraph, simulate_deferred
    from paper_2208_14567_b200.workloads import mixed_batch

    mb = mixed_batch(5000, 6, 8, seed=31, stride=8)
    p1 = torch.from_numpy(mb.pos).cuda()
    rng = np.random.default_rng(5)
    p2 = p1 + torch.from_numpy(rng.normal(0.0, 0.02, size=mb.pos.shape)).cuda()  # other poses, same topologies
    pos = p1.clone()
    topo = torch.from_numpy(mb.topo).cuda()
    table = mb.table()
    g = DeferredGraph(pos, table, 200, topo)
    for src in (p1, p2, p1):
        pos.copy_(src)
        out = g.replay()
        torch.cuda.synchronize()
        ref = simulate_deferred(src.clone(), table, 200, topo, dense_rows=True)
        for k in ("first_t", "first_joint"):
            assert torch.equal(out[k], ref[k]), k
        n = int(ref["pend_rows"].item())
        assert int(out["pend_rows"].item()) == n
        nv = int(ref["valid_count"].item())
        assert torch.equal(out["valid_idx"][:nv], ref["valid_idx"][:nv])
        np_ = int(ref["pend_count"].item())
        ok = (ref["first_t"][ref["pend_idx"][:np_]] == 200).cpu().numpy()
        rows = ref["pend_row"][:np_].cpu().numpy()
        nn = mb.n[ref["pend_idx"][:np_].cpu().numpy()]
        for i in np.flatnonzero(ok)[:500]:
            r0, r1 = int(rows[i]), int(rows[i] + nn[i])
            assert torch.equal(out["traj"][r0:r1], ref["traj"][r0:r1])


def test_bit_exact_f64_replay(torch, golden):
    """The f64 rounds follow numpy's operation order with IEEE ops and
    glibc's hypot: f64 paths are bit-identical to the reference, fp32 paths
    are the reference's values rounded once, and every lock flag (margin
    band included: those lanes are decided by the f64 replay) is exact."""
    from paper_2208_14567_b200.solver import SolutionPlan, compile_order
    from paper_2208_14567_b200.workloads import bare_plan, four_bar

    g = golden("solver_golden.npz")
    plan = bare_plan(four_bar())
    r64 = run_mixed(torch, [plan], g["fb_pos0"], None, 200, traj_f64=True)
    t64 = r64["traj"].view(-1, 4, 200, 2).cpu().numpy()
    assert np.array_equal(t64[g["fb_traj_idx"]], g["fb_traj"])
    assert np.array_equal(r64["first_t"].cpu().numpy(), g["fb_first_t"])
    assert np.array_equal(r64["first_joint"].cpu().numpy(), g["fb_first_joint"])
    plans = []
    for t in range(len(g["mx_n"])):
        n = int(g["mx_n"][t])
        fixed, steps = compile_order(g["mx_adj"][t][:n, :n], g["mx_types"][t][:n])
        plans.append(SolutionPlan(n, fixed, steps, None, None, None))
    for kw in ({}, {"fp64": True}):
        r32 = run_mixed(torch, plans, g["mx_pos0"], g["mx_topo"], 200, **kw)
        assert np.array_equal(r32["first_t"].cpu().numpy(), g["mx_first_t"])
        assert np.array_equal(r32["first_joint"].cpu().numpy(), g["mx_first_joint"])
        t32 = r32["traj"].view(-1, 20, 200, 2).cpu().numpy()
        r64 = run_mixed(torch, plans, g["mx_pos0"], g["mx_topo"], 200, traj_f64=True, **kw)
        t64 = r64["traj"].view(-1, 20, 200, 2).cpu().numpy()
        for gi, tp in zip(g["mx_traj_idx"], g["mx_traj"]):
            n = int(g["mx_n"][g["mx_topo"][gi]])
            assert np.array_equal(t64[gi, :n], tp[:n])
            assert np.array_equal(t32[gi, :n], tp[:n].astype(np.float32))


@pytest.mark.parametrize("seed", [901, 902])
def test_screen_flags_at_scale_vs_exact(torch, seed):
    """1M generator candidates of 5-20 joints: the fp32 screen's lock flags
    equal the all-f64 exact mode (bit-identical to the reference), except
    candidates whose oracle margin is inside the 1e-6 band (none expected).
    Long chains are where fp32 error amplification through flat dyads bites;
    the screen's error model (sim.cu solve32) must send those to f64."""
    from paper_2208_14567_b200.solver import simulate_tensors
    from paper_2208_14567_b200.workloads import native_batch

    nb = native_batch(1_000_000, 5, 20, seed=seed)
    pos = torch.from_numpy(nb.pos).cuda()
    topo = torch.from_numpy(nb.topo).cuda()
    ref = simulate_tensors(pos, nb.table, 200, topo, write_traj=False, fp64=True, exact=True)
    for kw in ({}, {"gate_only": True, "low": True}):
        res = simulate_tensors(pos, nb.table, 200, topo, write_traj=False, **kw)
        valid_ref = ref["first_t"] == 200
        if kw:
            bad = np.flatnonzero(((res["first_t"] == 200) != valid_ref).cpu().numpy())
        else:
            bad = np.flatnonzero(((res["first_t"] != ref["first_t"]) |
                                  (res["first_joint"] != ref["first_joint"])).cpu().numpy())
        raw = nb.table.host_bytes().reshape(-1, 64)
        for i in bad:
            rec = raw[int(nb.topo[i])]
            n = int(rec[0:2].view(np.int16)[0])
            ns = int(rec[2:4].view(np.int16)[0])
            fm = int(rec[4:8].view(np.uint32)[0])
            steps = [tuple(int(v) for v in s) for s in rec[8:8 + 3 * ns].astype(np.int8).reshape(ns, 3)]
            fixed = [k for k in range(n) if (fm >> k) & 1]
            m = O.simulate(nb.pos[i:i + 1, :n], steps, fixed, 200, with_margin=True)["margin"][0]
            assert m < MARGIN, f"candidate {i}: flag mismatch with margin {m:.3e} ({kw})"


def test_host_pipeline_matches_deferred(torch):
    """HostPipeline (chunked host-to-host pipeline, overlapped copies) returns
    the same flags, survivor ids and per-survivor paths as one
    DeferredGraph over the whole batch, for 1 and 3 chunks, with and without
    split rows (only dyad-target rows cross PCIe; HostPipeline.paths
    rebuilds the static joints and the crank tip bit-identical to the
    device's rows), and a second run over new host poses recomputes
    everything."""
    from paper_2208_14567_b200.solver import HostPipeline, simulate_deferred
    from paper_2208_14567_b200.workloads import mixed_batch

    mb = mixed_batch(4000, 6, 8, seed=37, stride=8)
    table = mb.table()
    pos_h = torch.from_numpy(mb.pos.copy())
    topo_h = torch.from_numpy(mb.topo)
    nsteps = np.array([len(p.steps) for p in mb.plans])[mb.topo]
    for chunks, split in ((1, True), (3, True), (3, False)):
        pipe = HostPipeline(pos_h, table, 200, topo_h, chunks=chunks, split_rows=split)
        for shift in (0.0, 0.01):
            pipe.pos_h.copy_(torch.from_numpy(mb.pos + shift))
            res = pipe.run()
            ref = simulate_deferred(pipe.pos_h.cuda(), table, 200, topo_h.cuda(), dense_rows=True)
            assert torch.equal(res["first_t"], ref["first_t"].cpu())
            assert torch.equal(res["first_joint"], ref["first_joint"].cpu())
            np_ = int(ref["pend_count"].item())
            assert torch.equal(res["pend_idx"], ref["pend_idx"][:np_].cpu())
            rr = ref["pend_row"][:np_].cpu().numpy()
            nn = mb.n[res["pend_idx"].numpy()]
            shipped = nsteps[res["pend_idx"].numpy()] if split else nn
            assert res["traj"].shape[0] == int(shipped.sum())
            assert res["d2h_bytes"] == 4000 * 8 + len(pipe.ranges) * 16 + int(shipped.sum()) * 200 * 8 + np_ * 16
            rt = ref["traj"].cpu().numpy()
            ok = (res["first_t"][res["pend_idx"]] == 200).numpy()  # rows of fine-pass locks are scratch
            for i in np.flatnonzero(ok)[::max(1, np_ // 300)]:
                assert np.array_equal(pipe.paths(res, int(i)), rt[rr[i]:rr[i] + nn[i]]), (chunks, split, i)


def test_split_rows_layout(torch):
    """simulate_deferred(split_rows=True): the dyad-target rows (traj) and the
    static + crank rows (traj2) of every valid survivor are the dense
    layout's rows, and assemble_paths' host rebuild of the static + crank
    rows is bit-identical to traj2 (numpy's crank arithmetic, np.hypot)."""
    from paper_2208_14567_b200.solver import assemble_paths, plan_row_split, simulate_deferred
    from paper_2208_14567_b200.workloads import mixed_batch

    mb = mixed_batch(6000, 5, 9, seed=41, stride=9)
    table = mb.table()
    pos, topo = torch.from_numpy(mb.pos).cuda(), torch.from_numpy(mb.topo).cuda()
    dense = simulate_deferred(pos, table, 200, topo, dense_rows=True)
    split = simulate_deferred(pos, table, 200, topo, split_rows=True)
    assert torch.equal(dense["first_t"], split["first_t"])
    np_ = int(dense["pend_count"].item())
    assert torch.equal(dense["pend_idx"][:np_], split["pend_idx"][:np_])
    idx = dense["pend_idx"][:np_].cpu().numpy()
    ft = dense["first_t"].cpu().numpy()
    dr, tr, orow = (dense["pend_row"][:np_].cpu().numpy(), split["pend_row"][:np_].cpu().numpy(),
                    split["pend_row2"][:np_].cpu().numpy())
    D, A, O2 = dense["traj"].cpu().numpy(), split["traj"].cpu().numpy(), split["traj2"].cpu().numpy()
    checked = 0
    for i, b in enumerate(idx):
        if ft[b] != 200:
            continue
        plan = mb.plans[mb.topo[b]]
        targets, others = plan_row_split(plan)
        full = D[dr[i]:dr[i] + plan.n]
        assert np.array_equal(A[tr[i]:tr[i] + len(targets)], full[targets])
        assert np.array_equal(O2[orow[i]:orow[i] + len(others)], full[others])
        assert np.array_equal(assemble_paths(A, int(tr[i]), mb.pos[b, :plan.n], plan.n, targets, 200), full)
        checked += 1
    assert checked > 500


def test_work_queue_schedule(torch):
    """The persistent grid's work queue (tickets of consecutive candidates)
    only changes which warp replays which candidate: flags, low-fidelity
    flags and paths equal the round-robin schedule (LA_SIM_STATIC_GRID) bit
    for bit, at sizes below one ticket per warp, around the chunking
    thresholds and with many tickets per warp; repeated launches on two
    streams (each takes its own counter pair, left zeroed by its kernel) keep
    returning the same answer."""
    from paper_2208_14567_b200 import _native as N
    from paper_2208_14567_b200.solver import simulate_tensors
    from paper_2208_14567_b200.workloads import native_batch

    nb = native_batch(400_000, 5, 20, seed=77)
    pos_all = torch.from_numpy(nb.pos).cuda()
    topo_all = torch.from_numpy(nb.topo).cuda()
    for count in (1, 33, 4_736, 40_001, 400_000):
        pos, topo = pos_all[:count], topo_all[:count]
        for kw in ({"write_traj": False}, {"write_traj": False, "gate_only": True, "low": True},
                   {"write_traj": True} if count <= 40_001 else None):
            if kw is None:
                continue
            # (zeroed path buffers: padding rows and the rows of locked
            # candidates past their first lock are not written)
            bufs = [dict(traj=torch.zeros((count * nb.table.max_n, 200, 2), dtype=torch.float32, device="cuda"))
                    if kw["write_traj"] else {} for _ in range(2)]
            ref = simulate_tensors(pos, nb.table, 200, topo, _extra_flags=N.LA_SIM_STATIC_GRID, **kw, **bufs[0])
            res = simulate_tensors(pos, nb.table, 200, topo, **kw, **bufs[1])
            for key in ref:
                assert torch.equal(ref[key], res[key]), (count, kw, key)
    pos, topo = pos_all[:100_000], topo_all[:100_000]
    ref = simulate_tensors(pos, nb.table, 200, topo, write_traj=False, _extra_flags=N.LA_SIM_STATIC_GRID)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for i in range(40):
        with torch.cuda.stream(streams[i % 2]):
            outs.append(simulate_tensors(pos, nb.table, 200, topo, write_traj=False, stream=streams[i % 2]))
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o["first_t"], ref["first_t"]) and torch.equal(o["first_joint"], ref["first_joint"])
