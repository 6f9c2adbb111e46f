"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference ``linkatlas`` package from
``/root/reference/pkg/src`` (read-only) and records its outputs on seeded
inputs.  The GPU box never runs this script; it only reads the committed
``.npz`` files.  Library versions are stored inside every fixture.
"""

from __future__ import annotations

import platform
import sys
from pathlib import Path

import numpy as np
import scipy

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

from linkatlas import atlas as ref_atlas  # noqa: E402
from linkatlas import curves as ref_curves  # noqa: E402
from linkatlas import generator as ref_gen  # noqa: E402
from linkatlas import solver as ref_solver  # noqa: E402
from linkatlas.mechanism import JointType, Mechanism  # noqa: E402

OUT = Path(__file__).resolve().parent
NMAX = 20
SMAX = 18


def versions():
    return np.array(
        f"python={platform.python_version()} numpy={np.__version__} scipy={scipy.__version__}"
    )


def four_bar(ground=(0.7, 0.5), coupler=(0.6, 0.62)) -> Mechanism:
    # same topology as the reference's tests/conftest.py:7-18 fixture
    adj = np.zeros((4, 4), dtype=np.uint8)
    for i, j in [(0, 1), (1, 3), (2, 3)]:
        adj[i, j] = adj[j, i] = 1
    types = np.array([0, 2, 0, 1], dtype=np.int8)
    pos = np.array([(0.5, 0.5), (0.55, 0.5), ground, coupler])
    return Mechanism(adj, types, pos)


def outcome_arrays(outs, T):
    ft = np.array([o.step if isinstance(o, ref_solver.Locking) else T for o in outs], dtype=np.int64)
    fj = np.array([o.joint if isinstance(o, ref_solver.Locking) else -1 for o in outs], dtype=np.int64)
    return ft, fj


def pack_topology(mech, plan):
    adj = np.zeros((NMAX, NMAX), dtype=np.uint8)
    adj[: mech.n, : mech.n] = mech.adjacency
    types = np.full(NMAX, -1, dtype=np.int8)
    types[: mech.n] = mech.types
    steps = np.full((SMAX, 3), -1, dtype=np.int16)
    for s, st in enumerate(plan.steps):
        steps[s] = (st.target, st.a, st.b)
    return adj, types, steps


def solver_fixture():
    d = {"versions": versions()}
    # --- C1-style four-bars
    mech = four_bar()
    plan = ref_solver.compile_plan(mech)
    rng = np.random.default_rng(0)
    pos = rng.uniform(size=(256, 4, 2))
    pos[:, 0] = (0.5, 0.5)
    pos[:, 1] = (0.55, 0.5)
    outs = ref_solver.simulate_batch(pos, plan, 200)
    ft, fj = outcome_arrays(outs, 200)
    d["fb_pos0"] = pos
    d["fb_first_t"] = ft
    d["fb_first_joint"] = fj
    valid = np.flatnonzero(ft == 200)[:12]
    d["fb_traj_idx"] = valid
    d["fb_traj"] = np.stack([outs[i].positions for i in valid])
    outs50 = ref_solver.simulate_batch(pos, plan, 50)
    d["fb_first_t50"], d["fb_first_joint50"] = outcome_arrays(outs50, 50)
    # --- known answers of the reference tests (test_solver.py:78-126)
    lock_mech = four_bar(ground=(0.9, 0.5), coupler=(0.72, 0.51))
    lp = ref_solver.compile_plan(lock_mech)
    o200 = ref_solver.simulate(lock_mech, lp, 200)
    o50 = ref_solver.simulate(lock_mech, lp, 50)
    d["ka_lock_pos0"] = lock_mech.positions0
    d["ka_lock"] = np.array([o200.step, o200.joint, o50.step, o50.joint])
    okm = four_bar()
    ok = ref_solver.simulate(okm, ref_solver.compile_plan(okm), 200)
    d["ka_valid_traj"] = ok.positions
    d["ka_dyad"] = np.array(ref_solver.dyad_solve((0.0, 0.0), (1.0, 0.0), 1.0, 1.0, 1.0))

    # --- mixed topologies from the reference generator (generator.py:200-238)
    adjs, typs, stps, ns, nsteps = [], [], [], [], []
    c_pos, c_topo, c_ft, c_fj, c_ft50, c_fj50 = [], [], [], [], [], []
    tr_idx, tr = [], []
    g = 0
    for n in [5, 6, 7, 8, 10, 12, 14, 16, 18, 20]:
        for rep in range(3):
            trng = np.random.default_rng([7, n, rep, 0])
            prng = np.random.default_rng([7, n, rep, 1])
            mech, plan = ref_gen.sample_topology(trng, n)
            a, t, s = pack_topology(mech, plan)
            adjs.append(a); typs.append(t); stps.append(s); ns.append(n); nsteps.append(len(plan.steps))
            cand = ref_gen._sample_positions_batch(n, 64, prng)
            outs = ref_solver.simulate_batch(cand, plan, 200)
            ft, fj = outcome_arrays(outs, 200)
            outs50 = ref_solver.simulate_batch(cand, plan, 50)
            ft50, fj50 = outcome_arrays(outs50, 50)
            padded = np.full((64, NMAX, 2), np.nan)
            padded[:, :n] = cand
            base = len(c_topo) * 1
            c_pos.append(padded); c_topo.append(np.full(64, g, dtype=np.int32))
            c_ft.append(ft); c_fj.append(fj); c_ft50.append(ft50); c_fj50.append(fj50)
            for i in np.flatnonzero(ft == 200)[:2]:
                tp = np.full((NMAX, 200, 2), np.nan)
                tp[:n] = outs[i].positions
                tr_idx.append(g * 64 + i)
                tr.append(tp)
            g += 1
    d["mx_adj"] = np.stack(adjs)
    d["mx_types"] = np.stack(typs)
    d["mx_steps"] = np.stack(stps)
    d["mx_n"] = np.array(ns, dtype=np.int32)
    d["mx_nsteps"] = np.array(nsteps, dtype=np.int32)
    d["mx_pos0"] = np.concatenate(c_pos)
    d["mx_topo"] = np.concatenate(c_topo)
    d["mx_first_t"] = np.concatenate(c_ft)
    d["mx_first_joint"] = np.concatenate(c_fj)
    d["mx_first_t50"] = np.concatenate(c_ft50)
    d["mx_first_joint50"] = np.concatenate(c_fj50)
    d["mx_traj_idx"] = np.array(tr_idx, dtype=np.int64)
    d["mx_traj"] = np.stack(tr)

    # --- find_valid_variant (generator.py:241-283): attempts + accepted pose
    fv_topo, fv_att, fv_pos, fv_seed = [], [], [], []
    for n, seed in [(6, 11), (8, 12), (8, 13), (10, 14), (12, 15)]:
        mech, plan = ref_gen.sample_topology(np.random.default_rng([seed, 0]), n)
        res = ref_gen.find_valid_variant(mech, plan, np.random.default_rng([seed, 1]))
        a, t, s = pack_topology(mech, plan)
        fv_topo.append((a, t, s, n))
        fv_att.append(res.attempts)
        p = np.full((NMAX, 2), np.nan)
        p[:n] = res.mechanism.positions0
        fv_pos.append(p)
        fv_seed.append(seed)
    d["fv_adj"] = np.stack([x[0] for x in fv_topo])
    d["fv_types"] = np.stack([x[1] for x in fv_topo])
    d["fv_steps"] = np.stack([x[2] for x in fv_topo])
    d["fv_n"] = np.array([x[3] for x in fv_topo], dtype=np.int32)
    d["fv_seed"] = np.array(fv_seed, dtype=np.int64)
    d["fv_attempts"] = np.array(fv_att, dtype=np.int64)
    d["fv_pos"] = np.stack(fv_pos)
    np.savez_compressed(OUT / "solver_golden.npz", **d)
    return d


def fourier_curves(seed: int, count: int, P: int) -> np.ndarray:
    """Random closed Fourier curves, 5 harmonics, coefficients N(0, 1/k^2)
    (BASELINE.json configs[3])."""
    rng = np.random.default_rng(seed)
    t = 2.0 * np.pi * np.arange(P) / P
    k = np.arange(1, 6)
    coef = rng.normal(size=(count, 4, 5)) / k
    cos_kt = np.cos(np.outer(t, k))  # (P, 5)
    sin_kt = np.sin(np.outer(t, k))
    x = coef[:, 0] @ cos_kt.T + coef[:, 1] @ sin_kt.T
    y = coef[:, 2] @ cos_kt.T + coef[:, 3] @ sin_kt.T
    return np.stack([x, y], axis=-1)


def curves_fixture(sol):
    d = {"versions": versions()}
    paths = []
    kinds = []
    # moving-joint curves of valid mixed mechanisms (cli.py:131-134 pattern)
    for tp, gi in zip(sol["mx_traj"], sol["mx_traj_idx"]):
        topo = sol["mx_topo"][gi]
        n = int(sol["mx_n"][topo])
        types = sol["mx_types"][topo]
        for j in range(n):
            if types[j] == 0:
                continue
            paths.append(tp[j]); kinds.append(0)
            if len(paths) >= 48:
                break
        if len(paths) >= 48:
            break
    for p in fourier_curves(5, 24, 200):
        paths.append(p); kinds.append(1)
    # reference-test style noisy lemniscates (test_curves.py:12-16)
    rng = np.random.default_rng(9)
    t = np.linspace(0, 2 * np.pi, 200, endpoint=False)
    for _ in range(8):
        p = np.stack([np.cos(t), np.sin(2 * t) * 0.4], axis=1) + rng.normal(scale=0.05, size=(200, 2))
        paths.append(p); kinds.append(2)
    # circle (is_circle true), and a scaled/shifted circle
    paths.append(np.stack([np.cos(t), np.sin(t)], axis=1) * 3.0 + 7.0); kinds.append(3)
    paths = np.stack(paths)
    outs, pairs, circ, circv, normd = [], [], [], [], []
    for p in paths:
        o = ref_curves.normalize(p)
        i, j, dd = ref_curves._farthest_pair(p)
        outs.append(o); pairs.append((i, j)); circ.append(ref_curves.is_circle(o))
        circv.append(float(np.var(np.hypot(o[:, 0] - 0.5, o[:, 1] - 0.5))))
        normd.append(ref_curves.is_normalized(o))
    d["paths"] = paths
    d["kinds"] = np.array(kinds, dtype=np.int8)
    d["normalized"] = np.stack(outs)
    d["pairs"] = np.array(pairs, dtype=np.int64)
    d["is_circle"] = np.array(circ)
    d["circle_var"] = np.array(circv)
    d["is_normalized"] = np.array(normd)
    d["is_normalized_raw"] = np.array([ref_curves.is_normalized(p) for p in paths])
    # the order-preservation example of SURVEY.md §8a a-7
    d["two_point"] = ref_curves.normalize(np.array([[2.0, 2.0], [4.0, 2.0]]))
    # chamfer pairs (curves.py:123-129) incl. known answer {(0,0)} vs {(1,0)}
    A = d["normalized"][:16]
    Bm = d["normalized"][16:32]
    d["chamfer_AB"] = np.array([[ref_curves.chamfer(a, b) for b in Bm] for a in A])
    d["chamfer_ka"] = np.array(ref_curves.chamfer(np.array([[0.0, 0.0]]), np.array([[1.0, 0.0]])))
    d["resample_64"] = np.stack([ref_curves.resample(p, 64) for p in paths[:4]])
    np.savez_compressed(OUT / "curves_golden.npz", **d)


def atlas_fixture():
    d = {"versions": versions()}
    N, P = 400, 64
    raw = fourier_curves(21, N, P)
    pts = np.stack([ref_curves.normalize(p) for p in raw])
    mech = four_bar()
    from linkatlas.records import CurveRecord

    recs = [CurveRecord(mech_id=i, joint_id=3, is_arc=False, is_circle=False, points=p.tolist())
            for i, p in enumerate(pts)]
    mechs = {i: mech for i in range(N)}
    atlas = ref_atlas.Atlas.build(recs, mechs, seed=3)
    assert np.array_equal(atlas.points, pts)
    d["points"] = pts
    d["order"] = atlas.order
    d["seed"] = np.array(3)
    queries = [
        pts[17].copy(),                                   # exact member -> self hit
        ref_curves.normalize(fourier_curves(99, 1, P)[0]),  # fresh curve
        ref_curves.normalize(fourier_curves(98, 1, P)[0]),
        ref_curves.normalize(np.array([[0.0, 0.0], [1.0, 1.0], [2.0, 0.0]])),  # far shape, Q=3
    ]
    cases = [(3, 0.03), (10, 1e-6), (5, 0.2), (3, np.inf)]
    rows = []
    for qi, q in enumerate(queries):
        for ci, (k, thr) in enumerate(cases):
            hits = atlas.retrieve(q, k=k, threshold=thr)
            for r, h in enumerate(hits):
                rows.append((qi, ci, r, h.mech_id, h.distance, float(h.above_threshold)))
    d["cases_k"] = np.array([c[0] for c in cases])
    d["cases_thr"] = np.array([c[1] for c in cases])
    d["hits"] = np.array(rows)
    for qi, q in enumerate(queries):
        d[f"query{qi}"] = q
        d[f"chamfer_cdist{qi}"] = np.array([ref_curves.chamfer(q, p) for p in pts])
        d[f"chamfer_block{qi}"] = ref_atlas._chamfer_block(pts, q)
    # brute-force ordering (test_atlas.py:106-118) for the fresh query
    full = atlas.retrieve(queries[1], k=N, threshold=np.inf)
    d["brute_ids"] = np.array([h.mech_id for h in full])
    d["brute_d"] = np.array([h.distance for h in full])
    # coarse prefilter (atlas.py:153-177): descriptors, filtered scan lists
    # and budgeted heuristic retrievals, on an atlas with duplicated curves
    # (tied descriptor distances) next to the plain one
    d["descriptors"] = atlas._build_descriptors()
    dup = np.concatenate([pts[:150], pts[:60], pts[100:130], pts[:60]])
    recs2 = [CurveRecord(mech_id=i, joint_id=3, is_arc=False, is_circle=False, points=p.tolist())
             for i, p in enumerate(dup)]
    atlas2 = ref_atlas.Atlas.build(recs2, {i: mech for i in range(len(dup))}, seed=11)
    d["dup_points"] = dup
    d["dup_order"] = atlas2.order
    d["dup_descriptors"] = atlas2._build_descriptors()
    budgets = [1, 7, 50, 61, 200]
    d["coarse_budgets"] = np.array(budgets)
    for qi, q in enumerate(queries + [pts[5].copy()]):
        d[f"coarse_q{qi}"] = q
        for bi, b in enumerate(budgets):
            d[f"coarse_{qi}_{bi}"] = atlas.coarse_filter(q, b)
            d[f"coarse_dup_{qi}_{bi}"] = atlas2.coarse_filter(q, b)
        hits = atlas2.retrieve(q, k=5, threshold=0.05, budget=61, filter_mode="heuristic")
        d[f"coarse_hits_{qi}"] = np.array([(h.mech_id, h.distance, float(h.above_threshold)) for h in hits])
    # Atlas.save (atlas.py:114-134) output bytes of a small atlas
    import tempfile

    small_recs = [CurveRecord(mech_id=i, joint_id=3, is_arc=False, is_circle=False, points=p.tolist())
                  for i, p in enumerate(pts[:12])]
    small = ref_atlas.Atlas.build(small_recs, {i: mech for i in range(12)}, seed=5)
    with tempfile.TemporaryDirectory() as tmp:
        small.save(tmp)
        for name in ("meta.json", "curves.ldjson", "mechanisms.ldjson"):
            d["save_" + name.replace(".", "_")] = np.frombuffer((Path(tmp) / name).read_bytes(), dtype=np.uint8)
    np.savez_compressed(OUT / "atlas_golden.npz", **d)


def generator_fixture():
    """GenerationRun (generator.py:336-375) records, stats and negatives."""
    d = {"versions": versions()}
    cases = [dict(count=30, seed=21), dict(count=12, seed=5, negative_rate=0.05),
             dict(count=20, seed=77, n_min=5, n_max=9, variants_per_topology=2, max_attempts=300)]
    for ci, kw in enumerate(cases):
        cfg = ref_gen.GenerationConfig(**kw)
        run = ref_gen.GenerationRun(cfg)
        recs = list(run.records())
        pos = np.full((len(recs), NMAX, 2), np.nan)
        meta = np.zeros((len(recs), 4), dtype=np.int64)  # slot, variant, attempts, n
        adj = np.zeros((len(recs), NMAX, NMAX), dtype=np.uint8)
        for i, r in enumerate(recs):
            n = r.mechanism.n
            pos[i, :n] = r.mechanism.positions0
            adj[i, :n, :n] = r.mechanism.adjacency
            meta[i] = (r.slot, r.variant, r.attempts, n)
        d[f"g{ci}_pos"] = pos
        d[f"g{ci}_meta"] = meta
        d[f"g{ci}_adj"] = adj
        d[f"g{ci}_traj_last"] = np.stack([r.trajectory.positions[-1] for r in recs])  # last joint path
        st = run.stats
        sizes = sorted(st.simulated_by_n)
        d[f"g{ci}_stats"] = np.array([[n, st.simulated_by_n.get(n, 0), st.accepted_by_n.get(n, 0)] for n in sizes])
        d[f"g{ci}_discarded"] = np.array(st.topologies_discarded)
        neg = np.full((len(run.negatives), NMAX, 2), np.nan)
        negstep = np.array([x.locking_step for x in run.negatives], dtype=np.int64)
        for i, x in enumerate(run.negatives):
            neg[i, :x.mechanism.n] = x.mechanism.positions0
        d[f"g{ci}_neg"] = neg
        d[f"g{ci}_negstep"] = negstep
        d[f"g{ci}_cfg"] = np.array([cfg.count, cfg.seed, cfg.n_min, cfg.n_max, cfg.variants_per_topology,
                                     cfg.T_low, cfg.T_high, cfg.max_attempts, cfg.batch, cfg.topology_retries])
        d[f"g{ci}_rates"] = np.array([cfg.ng_probability, cfg.negative_rate])
    # rejection_curve (generator.py:385-413)
    rc = ref_gen.rejection_curve(ref_gen.GenerationConfig(count=1, seed=7, max_attempts=1500), [6, 9, 12], trials=6)
    d["rc_sizes"] = np.array([6, 9, 12])
    d["rc_stats"] = np.array([[n, rc.simulated_by_n.get(n, 0), rc.accepted_by_n.get(n, 0)] for n in (6, 9, 12)])
    d["rc_samples"] = np.concatenate([np.array(rc.attempts_samples.get(n, []), dtype=np.int64) for n in (6, 9, 12)])
    np.savez_compressed(OUT / "generator_golden.npz", **d)


def dataset_fixture():
    """generate -> normalize -> curate chain of the CLI (cli.py:56-172):
    curve records of every moving joint, the keep rule, and the exact bytes
    of the reference's .ldjson writer for the kept curves and mechanisms."""
    import tempfile

    from linkatlas import records as ref_rec

    d = {"versions": versions()}
    cfg = ref_gen.GenerationConfig(count=24, seed=3, n_min=6, n_max=10, variants_per_topology=2, max_attempts=2000)
    recs = list(ref_gen.GenerationRun(cfg).records())
    curves, mrecs = [], []
    for rec in recs:
        mid = rec.slot * cfg.variants_per_topology + rec.variant
        mech = rec.mechanism
        mrecs.append(ref_rec.mechanism_to_record(mech, mid))
        for j in range(mech.n):
            if mech.types[j] == JointType.FIXED:
                continue
            pts = ref_curves.normalize(rec.trajectory.positions[j])
            curves.append(ref_rec.CurveRecord(mech_id=mid, joint_id=j, is_arc=ref_curves.is_arc(mech, j),
                                              is_circle=ref_curves.is_circle(pts), points=pts.tolist()))
    keep_rate, seed = 0.3, 4
    kept = list(ref_curves.curate(curves, keep_rate=keep_rate, seed=seed))
    d["cfg"] = np.array([cfg.count, cfg.seed, cfg.n_min, cfg.n_max, cfg.variants_per_topology, cfg.max_attempts])
    d["curate"] = np.array([keep_rate, seed])
    d["mech_ids"] = np.array([c.mech_id for c in curves])
    d["joint_ids"] = np.array([c.joint_id for c in curves])
    d["is_arc"] = np.array([c.is_arc for c in curves])
    d["is_circle"] = np.array([c.is_circle for c in curves])
    d["points"] = np.array([c.points for c in curves])
    d["kept"] = np.array([any(c is k for k in kept) for c in curves])
    with tempfile.TemporaryDirectory() as tmp:
        ref_rec.write_records(Path(tmp) / "c.ldjson", "curve", kept)
        ref_rec.write_records(Path(tmp) / "m.ldjson", "mechanism", mrecs)
        d["curves_ldjson"] = np.frombuffer((Path(tmp) / "c.ldjson").read_bytes(), dtype=np.uint8)
        d["mechs_ldjson"] = np.frombuffer((Path(tmp) / "m.ldjson").read_bytes(), dtype=np.uint8)
    # keep rule on wide ids (multi-word SeedSequence entropy)
    rng = np.random.default_rng(8)
    mids = np.concatenate([rng.integers(0, 2**31, 1000), rng.integers(2**32, 2**45, 1000), [0, 1, 2**32 - 1, 2**32]])
    jids = rng.integers(0, 20, len(mids))
    d["rule_mech"] = mids
    d["rule_joint"] = jids
    d["rule_keep"] = np.array([ref_curves.curation_keep(int(m), int(j), True, 0.5, 77) for m, j in zip(mids, jids)])
    np.savez_compressed(OUT / "dataset_golden.npz", **d)


def stream_fixture():
    """sample_topology's effect on the caller's stream (generator.py:200-222):
    two topologies drawn in sequence from one Generator, then the stream's
    next draws -- pins the RNG state the drop-in leaves behind."""
    d = {"versions": versions()}
    adj = np.zeros((24, 2, NMAX, NMAX), dtype=np.uint8)
    types = np.full((24, 2, NMAX), -1, dtype=np.int8)
    after = np.zeros((24, 3))
    ns = np.zeros(24, dtype=np.int32)
    for c in range(24):
        rng = np.random.default_rng([99, c])
        n = int(rng.integers(5, 21))
        ns[c] = n
        for k in range(2):
            mech, _ = ref_gen.sample_topology(rng, n)
            adj[c, k, :n, :n] = mech.adjacency
            types[c, k, :n] = mech.types
        after[c, :2] = rng.random(2)
        after[c, 2] = rng.integers(1000)
    d.update(adj=adj, types=types, after=after, n=ns)
    np.savez_compressed(OUT / "stream_golden.npz", **d)


if __name__ == "__main__" and sys.argv[1:] == ["stream"]:
    stream_fixture()
elif __name__ == "__main__":
    stream_fixture()
    sol = solver_fixture()
    curves_fixture(sol)
    atlas_fixture()
    generator_fixture()
    dataset_fixture()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
