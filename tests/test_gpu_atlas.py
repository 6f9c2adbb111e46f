"""GPU parity of the chamfer scan / retrieval against the reference atlas
fixture and the oracle; chamfer tolerance 1e-4 x bbox diagonal, top-k ids
equal except swaps between entries whose f64 distances differ by less than
that tolerance."""

import numpy as np
import pytest

from oracle import links_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def atlas_fx(golden):
    from paper_2208_14567_b200 import Atlas
    from paper_2208_14567_b200.workloads import four_bar

    g = golden("atlas_golden.npz")
    N = len(g["points"])
    mechs = {i: four_bar() for i in range(N)}
    atlas = Atlas(g["points"], np.arange(N), np.full(N, 3), mechs, seed=int(g["seed"]))
    return g, atlas


def ids_match(got_ids, got_d, want_ids, ref_d, tol=TOL):
    """Equal ids, allowing swaps among entries within tol of each other."""
    if len(got_ids) != len(want_ids):
        return False
    for a, b in zip(got_ids, want_ids):
        if a != b and abs(ref_d[a] - ref_d[b]) >= tol:
            return False
    return True


def test_order_and_exact_index(torch, atlas_fx):
    g, atlas = atlas_fx
    assert np.array_equal(atlas.order, g["order"])
    assert atlas.exact_index(g["points"][17]) == 17
    assert atlas.exact_index(g["query1"]) is None


def test_retrieve_matches_reference(torch, atlas_fx):
    g, atlas = atlas_fx
    hits = g["hits"]
    for qi in range(4):
        q = g[f"query{qi}"]
        ref_d = O.chamfer_direct_block(g["points"], q) if q.shape == g["points"].shape[1:] else \
            np.array([O.chamfer(q, p) for p in g["points"]])
        for ci, (k, thr) in enumerate(zip(g["cases_k"], g["cases_thr"])):
            want = hits[(hits[:, 0] == qi) & (hits[:, 1] == ci)]
            got = atlas.retrieve(q, k=int(k), threshold=float(thr))
            gid = [h.mech_id for h in got]
            wid = want[:, 3].astype(int).tolist()
            assert ids_match(gid, [h.distance for h in got], wid, ref_d), (qi, ci, gid, wid)
            for h, w in zip(got, want):
                assert abs(h.distance - w[4]) <= TOL
                if abs(ref_d[h.mech_id] - thr) > TOL:
                    assert h.above_threshold == bool(w[5])
                assert h.mechanism.n <= 4
    # self retrieval: exact 0.0 and not above threshold
    for i in [0, 200, 399]:
        h = atlas.retrieve(g["points"][i], k=1)
        assert h[0].distance == 0.0 and h[0].mech_id == i and not h[0].above_threshold


def test_brute_force_ordering(torch, atlas_fx):
    g, atlas = atlas_fx
    q = g["query1"]
    full = atlas.retrieve(q, k=len(atlas), threshold=np.inf)
    ref_d = O.chamfer_direct_block(g["points"], q)
    got = [h.mech_id for h in full]
    assert ids_match(got, None, g["brute_ids"].tolist(), ref_d)
    assert np.max(np.abs(np.array([h.distance for h in full]) - g["brute_d"])) <= TOL


def test_empty_and_padding(torch):
    from paper_2208_14567_b200 import Atlas

    a = Atlas(np.zeros((0, 0, 2)), np.zeros(0), np.zeros(0), {}, seed=0)
    assert a.retrieve(np.array([[0.0, 0.0], [1.0, 0.0]])) == []


def test_scan_topk_vs_oracle_large(torch):
    """Exhaustive top-10 over 200k Fourier curves (C4 shape) vs the oracle
    distances of the same fp32-stored curves."""
    from paper_2208_14567_b200.atlas import chamfer_scan
    from paper_2208_14567_b200.workloads import fourier_curves_device, fourier_db

    N, P = 200_000, 200
    db = fourier_db(N, P, seed=5, chunk=1 << 16)
    q = fourier_db(1, P, seed=77)[0]
    res = chamfer_scan(db, q[None], k=10, threshold=0.0, dense=True)
    torch.cuda.synchronize()
    dense = res["all_d"][0].cpu().numpy()
    top_id = res["top_id"][0].cpu().numpy()
    top_d = res["top_d"][0].cpu().numpy()
    # top list equals the ordering of the dense distances
    want = np.lexsort((np.arange(N), dense))[:10]
    assert np.array_equal(top_id, want)
    assert np.array_equal(top_d, dense[want])
    # oracle on a subset: the top-10 plus 2000 random records
    dbh = db.cpu().numpy().astype(np.float64)
    qh = q.cpu().numpy().astype(np.float64)
    sub = np.unique(np.concatenate([want, np.random.default_rng(0).choice(N, 2000, replace=False)]))
    ref = O.chamfer_direct_block(dbh[sub], qh)
    assert np.max(np.abs(dense[sub] - ref)) <= TOL
    assert int(res["n_hits"][0].item()) == 0


def test_scan_threshold_mode_and_shards(torch):
    """Threshold mode (first hits in scan order + padding) and the
    shard decomposition used by the multi-GPU merge give the same answer
    as one scan over everything."""
    from paper_2208_14567_b200.atlas import chamfer_scan
    from paper_2208_14567_b200.dist import local_scan_plan, merge_gathered, pack_lists
    from paper_2208_14567_b200.workloads import fourier_db

    N, P = 30_000, 64
    db = fourier_db(N, P, seed=9, chunk=1 << 14)
    qs = fourier_db(3, P, seed=10)
    order = np.random.default_rng(4).permutation(N)
    dorder = torch.from_numpy(order).cuda()
    res = chamfer_scan(db, qs, k=7, threshold=0.25, order=dorder, dense=True)
    dense = res["all_d"].cpu().numpy()
    pos_of = np.empty(N, dtype=np.int64)
    pos_of[order] = np.arange(N)
    for qi in range(3):
        d = dense[qi]
        hit = np.flatnonzero(d < 0.25)
        hit = hit[np.argsort(pos_of[hit])][:7]
        assert np.array_equal(res["hit_id"][qi].cpu().numpy()[: len(hit)], hit)
        non = np.flatnonzero(d >= 0.25)
        non = non[np.lexsort((pos_of[non], d[non]))][:7]
        assert np.array_equal(res["top_id"][qi].cpu().numpy(), non)
        assert int(res["n_hits"][qi].item()) == int((d < 0.25).sum())
    # 3 "ranks": contiguous record shards, global scan positions
    parts = []
    for r in range(3):
        lo, hi = r * N // 3, (r + 1) * N // 3
        lorder, pmap = local_scan_plan(order, lo, hi)
        parts.append(chamfer_scan(db[lo:hi], qs, k=7, threshold=0.25, order=torch.from_numpy(lorder).cuda(),
                                  pos_map=torch.from_numpy(pmap).cuda(), id_base=lo))
    merged = merge_gathered(torch.stack([pack_lists(p, 7) for p in parts]), 7)  # la_merge_shard_lists
    for name in ("top_d", "top_id", "hit_id", "top_pos", "hit_pos", "n_hits"):
        assert torch.equal(merged[name], res[name]), name


def test_retrieve_large_k_and_budget(torch, atlas_fx):
    g, atlas = atlas_fx
    q = g["query2"]
    ref = O.retrieve(g["points"], g["order"], q, 40, 0.25)
    got = atlas.retrieve(q, k=40, threshold=0.25)
    ref_d = O.chamfer_direct_block(g["points"], q)
    assert ids_match([h.mech_id for h in got], None, [r[1] for r in ref], ref_d)
    assert [h.above_threshold for h in got] == [bool(r[2]) for r in ref] or \
        any(abs(ref_d[r[1]] - 0.25) < TOL for r in ref)
    # budgeted scan with the heuristic prefilter only visits the filtered set
    # (the default filter_mode "exact" scans everything, atlas.py:157-158)
    hits = atlas.retrieve(q, k=3, budget=50, filter_mode="heuristic")
    allowed = set(atlas.coarse_filter(q, 50, "heuristic").tolist())
    assert len(allowed) == 50 and len(hits) == 3
    assert all(h.mech_id in allowed for h in hits)
    full = atlas.retrieve(q, k=3, budget=50)
    assert [h.mech_id for h in full] == [h.mech_id for h in atlas.retrieve(q, k=3)]


def test_chamfer_multi_query_and_odd_sizes(torch):
    from paper_2208_14567_b200.atlas import chamfer_scan

    rng = np.random.default_rng(3)
    for P, Q in ((199, 200), (64, 31), (256, 256), (9, 5)):
        db = rng.uniform(size=(500, P, 2)).astype(np.float32)
        qs = rng.uniform(size=(3, Q, 2)).astype(np.float32)
        res = chamfer_scan(torch.from_numpy(db).cuda(), torch.from_numpy(qs).cuda(), k=5, dense=True)
        d = res["all_d"].cpu().numpy()
        for qi in range(3):
            want = O.chamfer_direct_block(db.astype(np.float64), qs[qi].astype(np.float64))
            assert np.max(np.abs(d[qi] - want)) <= 1e-4
            top = np.lexsort((np.arange(500), d[qi]))[:5]
            assert res["top_id"][qi].tolist() == top.tolist()


def test_chamfer_many_queries_equal_single_scans(torch):
    """The wave-filling grid for many queries (CTAs per query chosen from
    the occupancy so the whole grid fills whole waves) returns, per query,
    exactly the lists and distances of a single-query scan."""
    from paper_2208_14567_b200.atlas import chamfer_scan
    from paper_2208_14567_b200.workloads import fourier_db

    db = fourier_db(60_000, 200, seed=4100)
    for nq in (2, 7, 64):
        qs = fourier_db(nq, 200, seed=500 + nq)
        many = chamfer_scan(db, qs, k=10, dense=True)
        for qi in sorted({0, nq // 2, nq - 1}):
            one = chamfer_scan(db, qs[qi:qi + 1], k=10, dense=True)
            assert torch.equal(many["all_d"][qi], one["all_d"][0]), (nq, qi)
            for n in ("top_id", "top_pos", "top_d", "hit_id", "n_hits"):
                assert torch.equal(many[n][qi], one[n][0]), (nq, qi, n)


def test_chamfer_expansion_mode_bound(torch):
    """Expansion inner loop with the rigorous rounding bound: every distance
    within fix_tol of the direct-difference value, near-duplicates re-checked."""
    from paper_2208_14567_b200.atlas import chamfer_scan
    from paper_2208_14567_b200.workloads import fourier_db

    db = fourier_db(20000, 200, seed=12, chunk=1 << 14)
    q = db[:3].clone()
    q[1] += 1e-4  # near-duplicate of record 1
    a = chamfer_scan(db, q, k=4, dense=True, expansion=True, fix_tol=5e-5)["all_d"].cpu().numpy()
    b = chamfer_scan(db, q, k=4, dense=True, expansion=False)["all_d"].cpu().numpy()
    assert np.max(np.abs(a - b)) <= 5e-5 + 1e-6
    assert a[0, 0] == 0.0 and a[2, 2] == 0.0


def test_chamfer_tensor_core_path(torch):
    """LA_CH_TENSOR (tcgen05 3xTF32 squared distances + direct recheck of
    small minima) agrees with the direct-difference kernel within the 1e-4
    tolerance, returns exact zeros for duplicated curves and the same top-k
    records on a Fourier database with planted duplicates."""
    from paper_2208_14567_b200.atlas import chamfer_scan
    from paper_2208_14567_b200.workloads import fourier_db

    db = fourier_db(20_000, 200, seed=4001)
    q = fourier_db(3, 200, seed=998)
    db[5] = q[0]
    db[17] = q[0]
    for P, Q in ((200, 200), (64, 200), (200, 37), (128, 128)):
        d_ = db[:, :P].contiguous()
        q_ = q[:, :Q].contiguous()
        a = chamfer_scan(d_, q_, k=10, dense=True)
        b = chamfer_scan(d_, q_, k=10, dense=True, tensor=True)
        da, dt = a["all_d"].cpu().numpy(), b["all_d"].cpu().numpy()
        assert np.max(np.abs(da - dt)) <= 1e-4, (P, Q)
        if P == 200 and Q == 200:
            assert dt[0, 5] == 0.0 and dt[0, 17] == 0.0
        # same records up to swaps of entries closer than the tolerance
        for qi in range(3):
            ia, ib = a["top_id"][qi].cpu().numpy(), b["top_id"][qi].cpu().numpy()
            for x, y in zip(ia, ib):
                if x != y:
                    assert abs(da[qi, x] - da[qi, y]) <= 2e-4
    # thresholded hits and an excluded record
    a = chamfer_scan(db, q, k=5, threshold=0.08, exclude_id=5)
    b = chamfer_scan(db, q, k=5, threshold=0.08, exclude_id=5, tensor=True)
    assert torch.equal(a["n_hits"], b["n_hits"])
    assert torch.equal(a["hit_id"], b["hit_id"])


def _lists_equal(torch, a, b, names=("top_d", "top_id", "top_pos", "hit_d", "hit_id", "hit_pos", "n_hits")):
    for name in names:
        assert torch.equal(a[name], b[name]), name


def test_pruned_scan_equals_full_scan(torch):
    """Exact pruning (query distance-grid lower bound vs the running k-th
    best) returns the same lists as evaluating every curve: C4-shaped
    single query, several queries with a shuffled order, hits, an excluded
    record and P = Q = 64, a scan order sorted worst-first (useless seed),
    and exact ties at the k-th place (copies of one curve)."""
    from paper_2208_14567_b200.atlas import chamfer_scan
    from paper_2208_14567_b200.workloads import fourier_db

    N, P = 300_000, 200
    db = fourier_db(N, P, seed=21, chunk=1 << 16)
    q = fourier_db(4, P, seed=22)
    full = chamfer_scan(db, q[:1], k=10, prune=False)
    pr = chamfer_scan(db, q[:1], k=10)
    _lists_equal(torch, full, pr)
    dense = chamfer_scan(db, q[:1], k=10, dense=True)["all_d"][0].cpu().numpy()
    assert np.array_equal(pr["top_id"][0].cpu().numpy(), np.lexsort((np.arange(N), dense))[:10])
    # several queries, shuffled order, threshold with hits, excluded record
    order = torch.from_numpy(np.random.default_rng(3).permutation(N)).cuda()
    thr = float(np.quantile(dense, 2e-5))
    ex = int(np.argmin(dense))
    kw = dict(k=7, threshold=thr, order=order, exclude_id=ex)
    _lists_equal(torch, chamfer_scan(db, q, prune=False, **kw), chamfer_scan(db, q, **kw))
    # worst-first scan order
    worst = torch.from_numpy(np.argsort(-dense, kind="stable")).cuda()
    _lists_equal(torch, chamfer_scan(db, q[:1], k=10, order=worst, prune=False),
                 chamfer_scan(db, q[:1], k=10, order=worst))
    # exact ties at the k-th place: 25 copies of the 3rd best curve
    third = int(np.lexsort((np.arange(N), dense))[2])
    dbt = db.clone()
    pos = np.random.default_rng(8).choice(N, 25, replace=False)
    dbt[torch.from_numpy(pos).cuda()] = db[third]
    a, b = chamfer_scan(dbt, q[:1], k=10, prune=False), chamfer_scan(dbt, q[:1], k=10)
    _lists_equal(torch, a, b)
    assert int((a["top_d"][0] == a["top_d"][0, 9]).sum().item()) >= 2
    # P = Q = 64 (other query register layout)
    db64 = fourier_db(100_000, 64, seed=23, chunk=1 << 16)
    q64 = fourier_db(3, 64, seed=24)
    _lists_equal(torch, chamfer_scan(db64, q64, k=10, prune=False), chamfer_scan(db64, q64, k=10))


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["expansion", "scalar_pipe", "odd_p", "seed_scan", "outside_unit_square"])
def test_pruned_scan_equals_full_scan_variants(torch, variant):
    """The pruning exactness argument (lb_slack covering fixup_below in
    expansion mode, the (1 - 1e-4) factor covering sqrt.approx and the fp16
    distance grid) across the inner-loop variants, an odd P (the non-TMA
    curve load), the seed prefix scan, and curves/queries partly outside
    [0, 1]^2 (clamped grid vertices)."""
    from paper_2208_14567_b200.atlas import chamfer_scan
    from paper_2208_14567_b200.workloads import fourier_db

    P = 199 if variant == "odd_p" else 200
    N = 200_000
    db = fourier_db(N, P, seed=31, chunk=1 << 16)
    q = fourier_db(3, P, seed=32)
    kw = {}
    if variant == "expansion":
        kw["expansion"] = True
    elif variant == "scalar_pipe":
        kw["scalar_pipe"] = True
    elif variant == "seed_scan":
        kw["seed_scan"] = True
    elif variant == "outside_unit_square":
        # stretch a third of the database and one query well past the unit box
        g = torch.Generator(device="cuda")
        g.manual_seed(5)
        sel = torch.randperm(N, device="cuda", generator=g)[: N // 3]
        db[sel] = (db[sel] - 0.5) * 2.5 + 0.5
        q[1] = (q[1] - 0.5) * 1.7 + torch.tensor([0.9, -0.4], device="cuda")
    full = chamfer_scan(db, q, k=10, prune=False, **kw)
    pr = chamfer_scan(db, q, k=10, **kw)
    _lists_equal(torch, full, pr)
    assert int(pr["n_full"].sum().item()) < 3 * N  # pruning did engage


@pytest.mark.parametrize("case", ["many_queries", "groups_hits_order", "expansion", "odd_q", "fine_grid",
                                  "outside_unit_square"])
def test_multi_query_scan_equals_unpruned(torch, case):
    """The multi-query pruned kernel (query groups sharing each streamed
    curve, box/gap-table column bound, common-grid row bound, then the
    single-query stages) returns the unpruned scan's lists: 64 queries,
    more queries than one group holds (hits, shuffled order, excluded
    record, pos_map), expansion mode, an odd query length (tail register
    slot), the 64x64 common grid, and data partly outside [0, 1]^2."""
    from paper_2208_14567_b200.atlas import chamfer_scan
    from paper_2208_14567_b200.workloads import fourier_db

    N, P = 120_000, 200
    db = fourier_db(N, P, seed=41, chunk=1 << 16)
    nq = 150 if case == "groups_hits_order" else 64
    q = fourier_db(nq, P, seed=42)
    kw = dict(k=10)
    if case == "groups_hits_order":
        dense = chamfer_scan(db, q[:1], k=10, dense=True)["all_d"][0].cpu().numpy()
        kw.update(k=6, threshold=float(np.quantile(dense, 1e-4)), exclude_id=int(np.argmin(dense)),
                  order=torch.from_numpy(np.random.default_rng(5).permutation(N)).cuda(),
                  pos_map=torch.arange(N, device="cuda", dtype=torch.int64) * 3 + 7)
    elif case == "expansion":
        kw["expansion"] = True
    elif case == "odd_q":
        q = q[:, :133].contiguous()
    elif case == "fine_grid":
        kw["mq_fine"] = True
    elif case == "outside_unit_square":
        g = torch.Generator(device="cuda")
        g.manual_seed(7)
        sel = torch.rand(N, generator=g, device="cuda") < 0.3
        db = db.clone()
        db[sel] = db[sel] * 1.7 - 0.35
        q = q.clone()
        q[:5] = q[:5] * 1.5 - 0.25
    mq = chamfer_scan(db, q, **kw)
    assert int(mq["n_stage"][0].item()) > 0  # the multi-query kernel ran
    _lists_equal(torch, chamfer_scan(db, q, prune=False, **{k: v for k, v in kw.items() if k != "mq_fine"}), mq)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c4", "order_hits_exclude", "odd_p", "outside_unit_square", "ties", "sharded",
                                  "expansion"])
def test_indexed_scan_equals_full_scan(torch, case):
    """Indexed single-query scans (la_chamfer_index cells: seed scan, bound
    step on the 2-byte cell rows, pruned scan of the survivors) return the
    lists of the scan that evaluates every curve: C4 shape; shuffled order
    with hits and an excluded record; odd P (16-bit cell loads); curves and
    query partly outside the unit square (border cells); exact ties at the
    k-th place; a shard with global positions (pos_map, id_base); the
    expansion inner loop (its slack enters the bound)."""
    from paper_2208_14567_b200.atlas import chamfer_index, chamfer_scan
    from paper_2208_14567_b200.workloads import fourier_db

    P = 199 if case == "odd_p" else 200
    N = 300_000
    db = fourier_db(N, P, seed=41, chunk=1 << 16)
    q = fourier_db(2, P, seed=42)
    kw = dict(k=10)
    if case == "outside_unit_square":
        g = torch.Generator(device="cuda")
        g.manual_seed(5)
        sel = torch.randperm(N, device="cuda", generator=g)[: N // 3]
        db[sel] = (db[sel] - 0.5) * 2.5 + 0.5
        q[0] = (q[0] - 0.5) * 1.7 + torch.tensor([0.9, -0.4], device="cuda")
    dense = chamfer_scan(db, q[:1], k=10, dense=True)["all_d"][0].cpu().numpy()
    if case == "order_hits_exclude":
        kw = dict(k=7, threshold=float(np.quantile(dense, 2e-5)), exclude_id=int(np.argmin(dense)),
                  order=torch.from_numpy(np.random.default_rng(3).permutation(N)).cuda())
    elif case == "ties":
        third = int(np.lexsort((np.arange(N), dense))[2])
        pos = np.random.default_rng(8).choice(N, 25, replace=False)
        db[torch.from_numpy(pos).cuda()] = db[third].clone()
    elif case == "sharded":
        rng = np.random.default_rng(9)
        kw = dict(k=10, id_base=1_000_000, pos_map=torch.from_numpy(np.sort(rng.choice(10 * N, N, replace=False))).cuda(),
                  order=torch.from_numpy(rng.permutation(N)).cuda())
    elif case == "expansion":
        kw = dict(k=10, expansion=True)
    cells = chamfer_index(db)
    for qq in (q[:1], q[1:2]):
        full = chamfer_scan(db, qq, prune=False, **kw)
        idx = chamfer_scan(db, qq, cells=cells, **kw)
        _lists_equal(torch, full, idx)
        surv, surv2 = int(idx["n_stage"][0].item()), int(idx["n_stage"][1].item())
        assert 0 < surv2 <= surv < N, (surv, surv2)  # both levels of the bound step ran and pruned
        # the index's parts on their own: cells only, cells + 16 x 16 tables
        for part in (cells.cells, cells._replace(fine=None)):
            _lists_equal(torch, full, chamfer_scan(db, qq, cells=part, **kw))
    if case == "c4":
        assert np.array_equal(chamfer_scan(db, q[:1], cells=cells, k=10)["top_id"][0].cpu().numpy(),
                              np.lexsort((np.arange(N), dense))[:10])
        # cells of points: floor((x + 1/32) * 1024 / 17) clamped, x major, rows of 66
        pts = db[:1000].cpu().numpy().astype(np.float64)
        cx = np.clip(np.floor((pts[..., 0] + 1 / 32) * 1024 / 17), 0, 63)
        cy = np.clip(np.floor((pts[..., 1] + 1 / 32) * 1024 / 17), 0, 63)
        got = cells.cells[:1000, :P].cpu().numpy().astype(np.int64)
        assert cells.cells.shape[1] == 208 and bool((cells.cells[:, P:] == 64).all())  # row padding: the null cell
        # coarse distance tables: floor(160 x distance from the 16 x 16 cell's box to the curve), saturated
        g0 = -1 / 32 + np.arange(16) * (17 / 256)
        a = pts[:50]
        ex = np.maximum(np.maximum(g0[:, None, None] - a[None, :, :, 0], a[None, :, :, 0] - (g0 + 17 / 256)[:, None, None]), 0)
        ey = np.maximum(np.maximum(g0[:, None, None] - a[None, :, :, 1], a[None, :, :, 1] - (g0 + 17 / 256)[:, None, None]), 0)
        ex[0] = np.maximum(a[..., 0] - (g0[0] + 17 / 256), 0)
        ex[15] = np.maximum(g0[15] - a[..., 0], 0)
        ey[0] = np.maximum(a[..., 1] - (g0[0] + 17 / 256), 0)
        ey[15] = np.maximum(g0[15] - a[..., 1], 0)
        dd = np.sqrt(ex[:, None] ** 2 + ey[None, :] ** 2).min(-1)  # (16, 16, 50)
        want = np.minimum(np.floor(dd * 160), 255).transpose(2, 0, 1).reshape(50, 256)
        gotc = cells.coarse[:50].cpu().numpy().astype(np.int64)
        assert (np.abs(gotc - want) <= 1).all() and (gotc <= want).mean() > 0.99
        # the 32 x 32 tables the same way
        g0 = -1 / 32 + np.arange(32) * (17 / 512)
        ex = np.maximum(np.maximum(g0[:, None, None] - a[None, :, :, 0], a[None, :, :, 0] - (g0 + 17 / 512)[:, None, None]), 0)
        ey = np.maximum(np.maximum(g0[:, None, None] - a[None, :, :, 1], a[None, :, :, 1] - (g0 + 17 / 512)[:, None, None]), 0)
        ex[0] = np.maximum(a[..., 0] - (g0[0] + 17 / 512), 0)
        ex[31] = np.maximum(g0[31] - a[..., 0], 0)
        ey[0] = np.maximum(a[..., 1] - (g0[0] + 17 / 512), 0)
        ey[31] = np.maximum(g0[31] - a[..., 1], 0)
        dd = np.sqrt(ex[:, None] ** 2 + ey[None, :] ** 2).min(-1)
        want = np.minimum(np.floor(dd * 160), 255).transpose(2, 0, 1).reshape(50, 1024)
        gotf = cells.fine[:50].cpu().numpy().astype(np.int64)
        assert (np.abs(gotf - want) <= 1).all() and (gotf <= want).mean() > 0.99
        assert (got == (cx * 66 + cy).astype(np.int64)).mean() > 0.999  # fp32 rounding at cell edges aside


@pytest.mark.gpu
def test_atlas_retrieve_with_cell_index(torch):
    """Atlas.retrieve on 80k stored curves (large enough for the pruned scan,
    so the atlas' cell index is used): the hits equal those of the same
    retrieval with the index disabled, for a stored curve (self hit), a
    fresh query, thresholds with and without hits, and the oracle's
    distances on the returned records."""
    import paper_2208_14567_b200.atlas as A
    from paper_2208_14567_b200 import Atlas
    from paper_2208_14567_b200.workloads import four_bar, fourier_db

    N = 80_000
    pts = fourier_db(N + 1, 200, seed=51, chunk=1 << 16).cpu().numpy().astype(np.float64)
    mech = four_bar()
    atlas = Atlas(pts[:N], np.arange(N), np.full(N, 3), {i: mech for i in range(N)}, seed=5)
    qs = [pts[123], pts[N]]
    dense = O.chamfer_direct_block(pts[:N], pts[N])
    for q in qs:
        for k, thr in ((10, 0.0), (5, float(np.quantile(dense, 1e-4)))):
            got = atlas.retrieve(q, k=k, threshold=thr)
            cells = atlas._cells_dev
            assert cells is not None and tuple(cells.cells.shape) == (N, 208) and tuple(cells.coarse.shape) == (N, 256)
            real = A.chamfer_scan

            def no_index(*a, **kw):
                kw["cells"] = None
                return real(*a, **kw)

            A.chamfer_scan = no_index
            try:
                want = atlas.retrieve(q, k=k, threshold=thr)
            finally:
                A.chamfer_scan = real
            assert [(h.mech_id, h.joint_id, h.distance, h.above_threshold) for h in got] == \
                   [(h.mech_id, h.joint_id, h.distance, h.above_threshold) for h in want]
            assert len(got) == k
    got = atlas.retrieve(pts[N], k=10, threshold=0.0)
    assert np.allclose(sorted(h.distance for h in got), np.sort(dense)[:10], atol=1e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["many_queries", "order_hits_exclude", "sharded", "odd_groups"])
def test_indexed_multi_query_scan_equals_full_scan(torch, case):
    """Indexed scans with several queries (multi-query seed, bound step with
    interleaved tables, per-query survivor lists): lists equal to evaluating
    every curve, with 40 queries (three groups of 16, the last partial), a
    shuffled order + hits + an excluded record, shard positions, and 17
    queries (a group of one)."""
    from paper_2208_14567_b200.atlas import chamfer_index, chamfer_scan
    from paper_2208_14567_b200.workloads import fourier_db

    N, P = 200_000, 200
    db = fourier_db(N, P, seed=61, chunk=1 << 16)
    nq = {"many_queries": 40, "odd_groups": 17}.get(case, 5)
    q = fourier_db(nq, P, seed=62)
    kw = dict(k=10)
    if case == "order_hits_exclude":
        dense = chamfer_scan(db, q[:1], k=10, dense=True)["all_d"][0].cpu().numpy()
        kw = dict(k=7, threshold=float(np.quantile(dense, 2e-5)), exclude_id=int(np.argmin(dense)),
                  order=torch.from_numpy(np.random.default_rng(3).permutation(N)).cuda())
    elif case == "sharded":
        rng = np.random.default_rng(9)
        kw = dict(k=10, id_base=1_000_000, pos_map=torch.from_numpy(np.sort(rng.choice(10 * N, N, replace=False))).cuda(),
                  order=torch.from_numpy(rng.permutation(N)).cuda())
    full = chamfer_scan(db, q, prune=False, **kw)
    idx = chamfer_scan(db, q, cells=chamfer_index(db), index_mq=True, **kw)
    _lists_equal(torch, full, idx)
    surv = int(idx["n_stage"][0].item())
    assert 0 < surv < nq * N, surv
