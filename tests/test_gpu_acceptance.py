"""End-to-end acceptance on the GPU pipeline, modelled on the reference's
desk-scale acceptance suite (pkg/tests/test_acceptance.py): a 42,000-record
corpus from GenerationRun, moving-joint curves normalised on the device,
arc/circle flags, the record-keyed curation rule, 64-point resampled atlas,
fresh queries.  Same thresholds as the reference's checks; the reference
suite takes about an hour on CPU, this one seconds.

Tolerances: f64 paths and normalisation are bit-exact with the reference
(LA_SIM_EXACT64, f64 la_normalize), so the 1e-9 / 1e-12 bars carry over;
retrieval distances come from the fp32 chamfer kernel (1e-4, north_star).
"""

import numpy as np
import pytest

from oracle import links_oracle as O

pytestmark = pytest.mark.gpu

CORPUS_COUNT = 42_000
CORPUS_SEED = 202
QUERY_SEED = 4242
ATLAS_POINTS = 64
KEEP_RATE = 0.005


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


def _resample_idx(P, count):
    return np.linspace(0, P - 1, count).round().astype(np.int64)


@pytest.fixture(scope="module")
def corpus(torch):
    from paper_2208_14567_b200.atlas import Atlas
    from paper_2208_14567_b200.curves import normalize_tensors
    from paper_2208_14567_b200.dataset import curation_keep_batch, curves_from_block, mechanisms_of_block
    from paper_2208_14567_b200.generator import GenerationConfig, GenerationRun

    cfg = GenerationConfig(count=CORPUS_COUNT, seed=CORPUS_SEED)
    run = GenerationRun(cfg, traj_on_device=True, lookahead=8)
    blocks = list(run.blocks())
    assert len(blocks) == 1
    blk = blocks[0]
    cb = curves_from_block(blk, cfg.variants_per_topology)
    flagged = cb.is_arc | cb.is_circle
    keep = curation_keep_batch(cb.mech_ids, cb.joint_ids, flagged, KEEP_RATE, CORPUS_SEED)
    kept = cb.select(keep)
    # resample to 64 of the path's own points, renormalise (f64, device)
    idx = torch.from_numpy(_resample_idx(kept.points.shape[1], ATLAS_POINTS)).cuda()
    small = normalize_tensors(kept.points.index_select(1, idx).contiguous(), out_f64=True)["out"]
    mechs = mechanisms_of_block(blk, cfg.variants_per_topology)
    atlas = Atlas(small.cpu().numpy(), kept.mech_ids, kept.joint_ids, mechs, CORPUS_SEED)
    # fresh queries (acceptance fixture: moving joint chosen by its own rng)
    qrun = GenerationRun(GenerationConfig(count=50, seed=QUERY_SEED))
    qrng = np.random.default_rng(QUERY_SEED)
    queries = []
    for rec in qrun.records():
        moving = [j for j in range(rec.mechanism.n) if rec.mechanism.types[j] != 0]
        j = int(qrng.choice(moving))
        p = O.normalize(rec.trajectory.positions[j])
        queries.append(O.normalize(O.resample(p, ATLAS_POINTS)))
    return dict(run=run, blk=blk, cb=cb, flagged=flagged, kept=kept, atlas=atlas, queries=queries,
                mechs=mechs, small=small)


def test_rejection_curve_matches_reference(torch, golden):
    from paper_2208_14567_b200.generator import GenerationConfig, rejection_curve

    g = golden("generator_golden.npz")
    st = rejection_curve(GenerationConfig(count=1, seed=7, max_attempts=1500), list(g["rc_sizes"]), trials=6)
    got = np.array([[n, st.simulated_by_n.get(n, 0), st.accepted_by_n.get(n, 0)] for n in g["rc_sizes"]])
    assert np.array_equal(got, g["rc_stats"])
    samples = np.concatenate([np.array(st.attempts_samples.get(int(n), []), dtype=np.int64) for n in g["rc_sizes"]])
    assert np.array_equal(samples, g["rc_samples"])


def test_solver_conservation(corpus):
    """Edge lengths conserved to 1e-9 over T = 200 on 1000 generated
    mechanisms; the scalar drop-in reproduces the batch paths exactly."""
    from paper_2208_14567_b200 import compile_plan, simulate

    blk = corpus["blk"]
    worst = 0.0
    for i in range(1000):
        rec = blk.record(i)
        mech, P = rec.mechanism, rec.trajectory.positions
        for a, b in mech.edges():
            d = np.hypot(*(P[a] - P[b]).T)
            worst = max(worst, float(d.max() - d.min()))
        if i < 100:
            out = simulate(mech, compile_plan(mech), 200)
            assert np.array_equal(out.positions, P)
    assert worst < 1e-9


def test_four_bar_against_independent_rootfinder(torch):
    """100 feasible random four-bars: positions match a loop-closure
    root-finder (scipy fsolve) to 1e-6 (acceptance: four-bar oracle)."""
    from scipy.optimize import fsolve

    from paper_2208_14567_b200 import Locking, compile_plan, simulate
    from paper_2208_14567_b200.workloads import four_bar

    rng = np.random.default_rng(99)
    checked, worst = 0, 0.0
    while checked < 100:
        mech = four_bar(ground=tuple(rng.uniform([0.55, 0.3], [0.95, 0.7])),
                        coupler=tuple(rng.uniform([0.4, 0.4], [0.85, 0.85])))
        out = simulate(mech, compile_plan(mech), 100)
        if isinstance(out, Locking):
            continue
        checked += 1
        p0, p2 = mech.positions0[0], mech.positions0[2]
        r2 = np.linalg.norm(mech.positions0[3] - mech.positions0[1])
        r4 = np.linalg.norm(mech.positions0[3] - p2)
        g = p2 - p0
        v3 = mech.positions0[3] - mech.positions0[1]
        v4 = mech.positions0[3] - p2
        guess = np.array([np.arctan2(v3[1], v3[0]), np.arctan2(v4[1], v4[0])])
        for t in range(100):
            th = 2 * np.pi * t / 100
            crank = 0.05 * np.array([np.cos(th), np.sin(th)])

            def closure(x, crank=crank):
                return (crank + r2 * np.array([np.cos(x[0]), np.sin(x[0])]) - g
                        - r4 * np.array([np.cos(x[1]), np.sin(x[1])]))

            sol, _, ier, _ = fsolve(closure, guess, full_output=True)
            assert ier == 1
            guess = sol
            expect = p0 + crank + r2 * np.array([np.cos(sol[0]), np.sin(sol[0])])
            worst = max(worst, float(np.linalg.norm(out.positions[3, t] - expect)))
    assert worst < 1e-6


def test_bias_statistic_and_curation(corpus):
    """Arc-or-circle fraction 62 +/- 15 % on >= 1e5 uncurated curves; under
    2 % after the 0.5 % keep-rate curation."""
    cb, flagged, kept = corpus["cb"], corpus["flagged"], corpus["kept"]
    assert len(cb) >= 100_000
    frac = flagged.mean()
    assert 0.47 <= frac <= 0.77
    assert (kept.is_arc | kept.is_circle).mean() < 0.02


def test_normalization_properties(torch, corpus):
    """Idempotence and similarity invariance over 1e4 random transforms at
    1e-9 (frame-stable bases), unit diameter and box centre — the whole
    batch in one f64 la_normalize launch."""
    from paper_2208_14567_b200.curves import normalize_tensors

    rng = np.random.default_rng(17)
    pts = corpus["small"].cpu().numpy()

    def stable(p):
        d = np.sqrt(((p[:, None] - p[None, :]) ** 2).sum(-1))
        return int((d > d.max() * (1.0 - 1e-7)).sum()) == 2

    bases = []
    while len(bases) < 100:
        c = pts[int(rng.integers(len(pts)))]
        if stable(c):
            bases.append(c)
    canon = normalize_tensors(torch.from_numpy(np.stack(bases)).cuda(), out_f64=True)["out"]
    again = normalize_tensors(canon, out_f64=True)["out"]
    assert float((again - canon).abs().max()) < 1e-9
    cn = canon.cpu().numpy()
    for c in cn:
        d = np.sqrt(((c[:, None] - c[None, :]) ** 2).sum(-1)).max()
        assert abs(d - 1.0) < 1e-12
        assert np.allclose((c.min(axis=0) + c.max(axis=0)) / 2, [0.5, 0.5], atol=1e-12)
    moved = []
    for base in bases:
        for _ in range(100):
            ang = rng.uniform(0, 2 * np.pi)
            scale = np.exp(rng.uniform(np.log(0.05), np.log(20.0)))
            shift = rng.uniform(-30, 30, size=2)
            c, s = np.cos(ang), np.sin(ang)
            moved.append(scale * base @ np.array([[c, -s], [s, c]]).T + shift)
    out = normalize_tensors(torch.from_numpy(np.stack(moved)).cuda(), out_f64=True)["out"].cpu().numpy()
    out = out.reshape(100, 100, ATLAS_POINTS, 2)
    err = np.minimum(np.abs(out - cn[:, None]).max(axis=(2, 3)), np.abs((1.0 - out) - cn[:, None]).max(axis=(2, 3)))
    assert float(err.max()) < 1e-9


def test_retrieval_at_scale(torch, corpus):
    """>= 1e5-curve atlas: >= 40 % of 50 fresh queries get a sub-0.03 hit;
    members self-retrieve at 0; a 1e4-record atlas retrieves everything in
    the brute-force chamfer order (fp32 chamfer: 1e-4)."""
    from paper_2208_14567_b200.atlas import Atlas

    atlas = corpus["atlas"]
    assert len(atlas) >= 100_000
    found = 0
    for q in corpus["queries"]:
        hits = atlas.retrieve(q, k=3, threshold=0.03)
        found += bool(hits) and not hits[0].above_threshold
    assert found / len(corpus["queries"]) >= 0.40
    rng = np.random.default_rng(23)
    for i in rng.choice(len(atlas), size=20, replace=False):
        assert atlas.retrieve(atlas.points[i], k=1)[0].distance == 0.0
    kept = corpus["kept"]
    small = Atlas(atlas.points[:10_000], kept.mech_ids[:10_000], kept.joint_ids[:10_000], corpus["mechs"], seed=1)
    for q in corpus["queries"][:3]:
        brute = np.sort([O.chamfer(q, small.points[i]) for i in range(len(small))])
        got = np.array([h.distance for h in small.retrieve(q, k=len(small), threshold=np.inf)])
        assert np.allclose(got, brute, atol=1e-4)
