"""Pin the CPU oracle (oracle/links_oracle.py) against fixtures the reference
itself produced (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import links_oracle as O


def _steps(row, nsteps):
    return [tuple(int(v) for v in row[s]) for s in range(nsteps)]


def test_fourbar_flags_and_trajectories(golden):
    g = golden("solver_golden.npz")
    steps, fixed = O.compile_steps(
        np.array([[0, 1, 0, 0], [1, 0, 0, 1], [0, 0, 0, 1], [0, 1, 1, 0]]), [0, 2, 0, 1])
    assert fixed == (0, 2) and [s[0] for s in steps] == [3]
    res = O.simulate(g["fb_pos0"], steps, fixed, 200)
    assert np.array_equal(res["first_t"], g["fb_first_t"])
    assert np.array_equal(res["first_joint"], g["fb_first_joint"])
    P = O.trajectories(res)[g["fb_traj_idx"]]
    assert np.array_equal(P, g["fb_traj"])  # bit-exact f64 restatement
    r50 = O.simulate(g["fb_pos0"], steps, fixed, 50)
    assert np.array_equal(r50["first_t"], g["fb_first_t50"])
    assert np.array_equal(r50["first_joint"], g["fb_first_joint50"])


def test_known_answers(golden):
    g = golden("solver_golden.npz")
    steps = [(3, 1, 2)]
    r = O.simulate(g["ka_lock_pos0"][None], steps, (0, 2), 200)
    assert (r["first_t"][0], r["first_joint"][0]) == tuple(g["ka_lock"][:2])
    r = O.simulate(g["ka_lock_pos0"][None], steps, (0, 2), 50)
    assert (r["first_t"][0], r["first_joint"][0]) == tuple(g["ka_lock"][2:])
    assert tuple(g["ka_lock"][:2]) == (5, 3) and g["ka_lock"][2] == 2
    ok = O.trajectories(O.simulate(g["ka_valid_traj"][:, 0, :][None], steps, (0, 2), 200))[0]
    assert np.array_equal(ok, g["ka_valid_traj"])
    assert np.allclose(g["ka_dyad"], (0.5, 0.8660254037844386), atol=0, rtol=0)


def test_mixed_topologies(golden):
    g = golden("solver_golden.npz")
    for topo in range(len(g["mx_n"])):
        n = int(g["mx_n"][topo])
        steps, fixed = O.compile_steps(g["mx_adj"][topo][:n, :n], g["mx_types"][topo][:n])
        assert steps == _steps(g["mx_steps"][topo], int(g["mx_nsteps"][topo]))
        sel = np.flatnonzero(g["mx_topo"] == topo)
        pos = g["mx_pos0"][sel][:, :n]
        r = O.simulate(pos, steps, fixed, 200)
        assert np.array_equal(r["first_t"], g["mx_first_t"][sel])
        assert np.array_equal(r["first_joint"], g["mx_first_joint"][sel])
        r50 = O.simulate(pos, steps, fixed, 50)
        assert np.array_equal(r50["first_t"], g["mx_first_t50"][sel])
        assert np.array_equal(r50["first_joint"], g["mx_first_joint50"][sel])
        P = O.trajectories(r)
        for gi, tp in zip(g["mx_traj_idx"], g["mx_traj"]):
            if g["mx_topo"][gi] == topo:
                assert np.array_equal(P[gi - sel[0]], tp[:n])


def test_t50_is_subset_of_t200(golden):
    """SURVEY probe P5: the 50-angle sweep equals every 4th angle of 200."""
    c200, s200 = O.crank_angles(200)
    c50, s50 = O.crank_angles(50)
    assert np.array_equal(c200[::4], c50) and np.array_equal(s200[::4], s50)


def test_normalize_matches_reference(golden):
    g = golden("curves_golden.npz")
    for p, want, pair, circ, var in zip(g["paths"], g["normalized"], g["pairs"],
                                        g["is_circle"], g["circle_var"]):
        i, j, _ = O.farthest_pair(p)
        assert (i, j) == tuple(pair)
        got = O.normalize(p)
        assert np.max(np.abs(got - want)) <= 1e-15
        assert O.is_circle(got) == bool(circ)
        assert abs(O.circle_variance(got) - var) <= 1e-15
    assert np.array_equal(O.normalize(np.array([[2.0, 2.0], [4.0, 2.0]])), g["two_point"])
    assert [O.is_normalized(x) for x in g["normalized"]] == list(g["is_normalized"])
    assert [O.is_normalized(x) for x in g["paths"]] == list(g["is_normalized_raw"])
    for p, r in zip(g["paths"][:4], g["resample_64"]):
        assert np.array_equal(O.resample(p, 64), r)


def test_normalize_errors():
    with pytest.raises(ValueError):
        O.normalize(np.full((10, 2), 0.3))
    with pytest.raises(ValueError):
        O.normalize(np.zeros((1, 2)))


def test_chamfer_matches_reference(golden):
    g = golden("curves_golden.npz")
    A, B = g["normalized"][:16], g["normalized"][16:32]
    got = np.array([[O.chamfer(a, b) for b in B] for a in A])
    assert np.max(np.abs(got - g["chamfer_AB"])) <= 1e-12
    assert O.chamfer(np.array([[0.0, 0.0]]), np.array([[1.0, 0.0]])) == float(g["chamfer_ka"]) == 2.0


def test_atlas_scan_matches_reference(golden):
    g = golden("atlas_golden.npz")
    pts, order = g["points"], g["order"]
    assert np.array_equal(np.random.default_rng(int(g["seed"])).permutation(len(pts)), order)
    hits = g["hits"]
    for qi in range(4):
        q = g[f"query{qi}"]
        if q.shape == pts.shape[1:]:
            blk = O.chamfer_expansion_block(pts, q)
            assert np.array_equal(blk, g[f"chamfer_block{qi}"])
            assert np.max(np.abs(O.chamfer_direct_block(pts, q) - g[f"chamfer_cdist{qi}"])) <= 1e-12
        for ci, (k, thr) in enumerate(zip(g["cases_k"], g["cases_thr"])):
            want = hits[(hits[:, 0] == qi) & (hits[:, 1] == ci)]
            got = O.retrieve(pts, order, q, int(k), float(thr))
            assert [r[1] for r in got] == want[:, 3].astype(int).tolist()
            assert np.array_equal(np.array([r[0] for r in got]), want[:, 4])
            assert [float(r[2]) for r in got] == want[:, 5].tolist()
    full = O.retrieve(pts, order, g["query1"], len(pts), np.inf)
    assert [r[1] for r in full] == g["brute_ids"].tolist()


def test_oracle_coarse_filter_pinned(golden):
    """Descriptors and heuristic scan lists equal the reference's, including
    an atlas with duplicated curves (tied descriptor distances)."""
    g = golden("atlas_golden.npz")
    desc = np.stack([O.coarse_descriptor(p) for p in g["points"]])
    assert np.array_equal(desc, g["descriptors"])
    ddesc = np.stack([O.coarse_descriptor(p) for p in g["dup_points"]])
    assert np.array_equal(ddesc, g["dup_descriptors"])
    budgets = g["coarse_budgets"]
    for qi in range(5):
        q = g[f"coarse_q{qi}"]
        qd = O.coarse_descriptor(q)
        for bi, b in enumerate(budgets):
            assert np.array_equal(O.coarse_filter(desc, g["order"], qd, int(b)), g[f"coarse_{qi}_{bi}"])
            assert np.array_equal(O.coarse_filter(ddesc, g["dup_order"], qd, int(b)), g[f"coarse_dup_{qi}_{bi}"])


def test_scalar_replay_matches_reference(golden):
    """oracle.simulate_scalar (solver.py:142-169) against the reference's
    batch outputs: lock (t, joint) and bit-exact f64 paths (the reference
    asserts scalar == batch bit for bit, solver.py:146-147)."""
    g = golden("solver_golden.npz")
    steps = [(3, 1, 2)]
    traj = dict(zip(g["fb_traj_idx"].tolist(), g["fb_traj"]))
    for b in range(64):
        kind, *rest = O.simulate_scalar(g["fb_pos0"][b], steps, (0, 2), 200)
        if kind == "lock":
            assert (rest[0], rest[1]) == (g["fb_first_t"][b], g["fb_first_joint"][b])
        else:
            assert g["fb_first_t"][b] == 200
            if b in traj:
                assert np.array_equal(rest[0], traj[b])
    for topo in range(0, len(g["mx_n"]), 7):
        n = int(g["mx_n"][topo])
        steps, fixed = O.compile_steps(g["mx_adj"][topo][:n, :n], g["mx_types"][topo][:n])
        sel = np.flatnonzero(g["mx_topo"] == topo)[:16]
        for b in sel:
            kind, *rest = O.simulate_scalar(g["mx_pos0"][b][:n], steps, fixed, 200)
            if kind == "lock":
                assert (rest[0], rest[1]) == (g["mx_first_t"][b], g["mx_first_joint"][b])
            else:
                assert g["mx_first_t"][b] == 200


def test_gate_matches_reference_sweeps(golden):
    """oracle.gate (generator.py:263-275 pattern): valid iff the reference's
    T=200 replay is lock-free; the T_low step is the reference's T=50 lock."""
    g = golden("solver_golden.npz")
    for topo in range(len(g["mx_n"])):
        n = int(g["mx_n"][topo])
        steps, fixed = O.compile_steps(g["mx_adj"][topo][:n, :n], g["mx_types"][topo][:n])
        sel = np.flatnonzero(g["mx_topo"] == topo)
        valid, low_t = O.gate(g["mx_pos0"][sel][:, :n], steps, fixed, 50, 200)
        assert np.array_equal(valid, g["mx_first_t"][sel] == 200)
        want_low = np.where(g["mx_first_t50"][sel] < 50, g["mx_first_t50"][sel], -1)
        assert np.array_equal(low_t, want_low)
