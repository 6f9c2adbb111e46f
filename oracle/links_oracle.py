"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference hot path.

Each function cites the reference ``linkatlas`` source it restates
(``/root/reference/pkg/src/linkatlas/<file>.py:<line>``).  The arithmetic is
float64 numpy in the same operation order as the reference so that, on the
same numpy build, results agree bit-for-bit (pinned by
``tests/test_oracle_golden.py`` against fixtures the reference produced).

Nothing in the product package may import this module.
"""

from __future__ import annotations

import numpy as np

LOCK_EPS = 1e-9                    # solver.py:19
CIRCLE_VARIANCE_THRESHOLD = 5e-4   # curves.py:14
NORM_TOL = 1e-9                    # curves.py:15
FIXED, SIMPLE, ACTUATED = 0, 1, 2  # mechanism.py:28-32


# ---------------------------------------------------------------- solve order
def compile_steps(adjacency: np.ndarray, types: np.ndarray):
    """Two-known-neighbours walk (solver.py:71-102).

    Returns (steps, fixed) with steps a list of (target, a, b).  Joints become
    known immediately inside a pass; unknowns are scanned in ascending order.
    Raises ValueError on a stall (the reference raises PlanError).
    """
    adj = np.asarray(adjacency)
    n = adj.shape[0]
    fixed = [k for k in range(n) if int(types[k]) == FIXED]
    known = set(fixed)
    known.add(1)
    pending = [k for k in range(n) if k not in known]
    steps = []
    while pending:
        advanced = False
        for k in list(pending):
            parents = [v for v in np.flatnonzero(adj[k]).tolist() if v in known]
            if len(parents) < 2:
                continue
            steps.append((k, parents[0], parents[1]))
            known.add(k)
            pending.remove(k)
            advanced = True
        if not advanced:
            raise ValueError(f"not dyadically solvable: {sorted(pending)}")
    return steps, tuple(fixed)


def step_geometry(pos0: np.ndarray, steps):
    """Per-candidate bar lengths and branch signs (solver.py:105-120, 189-201).

    pos0: (B, n, 2) float64.  Returns r_a, r_b, branch, each (B, S).
    """
    pos0 = np.asarray(pos0, dtype=np.float64)
    tg = np.array([s[0] for s in steps], dtype=np.intp)
    ia = np.array([s[1] for s in steps], dtype=np.intp)
    ib = np.array([s[2] for s in steps], dtype=np.intp)
    ax, ay = pos0[:, ia, 0], pos0[:, ia, 1]
    bx, by = pos0[:, ib, 0], pos0[:, ib, 1]
    tx, ty = pos0[:, tg, 0], pos0[:, tg, 1]
    r_a = np.hypot(tx - ax, ty - ay)
    r_b = np.hypot(tx - bx, ty - by)
    cross = (bx - ax) * (ty - ay) - (by - ay) * (tx - ax)
    branch = np.where(cross >= 0.0, 1.0, -1.0)
    return r_a, r_b, branch


def crank_angles(T: int):
    """theta_t = 2*pi*t/T and its cos/sin (solver.py:156-158, 180)."""
    th = 2.0 * np.pi * np.arange(T) / T
    return np.cos(th), np.sin(th)


def simulate(pos0: np.ndarray, steps, fixed, T: int = 200, with_margin: bool = False):
    """Batch replay of one plan (solver.py:172-239).

    Returns dict with X, Y (B, n, T) float64 (NaN where locked/unsolved),
    first_t (B,) int64 (T when valid), first_joint (B,) int64 (-1 when valid),
    and optionally ``margin`` (B,): min over steps and t <= first_t of the
    normalised discriminant |g| (SURVEY.md §8a parity rule), NaN-free.
    """
    pos0 = np.asarray(pos0, dtype=np.float64)
    B, n, _ = pos0.shape
    X = np.full((B, n, T), np.nan)
    Y = np.full((B, n, T), np.nan)
    still = sorted(set(fixed) | {0})
    X[:, still, :] = pos0[:, still, 0][:, :, None]
    Y[:, still, :] = pos0[:, still, 1][:, :, None]
    cos_t, sin_t = crank_angles(T)
    r1 = np.hypot(pos0[:, 1, 0] - pos0[:, 0, 0], pos0[:, 1, 1] - pos0[:, 0, 1])
    X[:, 1, :] = pos0[:, 0, 0, None] + r1[:, None] * cos_t[None, :]
    Y[:, 1, :] = pos0[:, 0, 1, None] + r1[:, None] * sin_t[None, :]

    first_t = np.full(B, T, dtype=np.int64)
    first_joint = np.full(B, -1, dtype=np.int64)
    gmin = np.full((B, T), np.inf)
    if steps:
        R_a, R_b, BR = step_geometry(pos0, steps)
    for s, (tg, a, b) in enumerate(steps):
        dx = X[:, b, :] - X[:, a, :]
        dy = Y[:, b, :] - Y[:, a, :]
        d = np.hypot(dx, dy)
        ra = R_a[:, s, None]
        rb = R_b[:, s, None]
        locked = (d < LOCK_EPS) | (d > ra + rb + LOCK_EPS) | (d < np.abs(ra - rb) - LOCK_EPS)
        with np.errstate(invalid="ignore", divide="ignore"):
            x = (d * d + ra * ra - rb * rb) / (2.0 * d)
            h = np.sqrt(np.maximum(ra * ra - x * x, 0.0))
            ux = dx / d
            uy = dy / d
            bh = BR[:, s, None] * h
            nx = X[:, a, :] + x * ux - bh * uy
            ny = Y[:, a, :] + x * uy + bh * ux
            if with_margin:
                sp = ra + rb
                g = np.minimum(sp * sp - d * d, d * d - (ra - rb) ** 2) / (sp * sp)
                g = np.where(np.isnan(g), np.inf, np.abs(g))
                gmin = np.minimum(gmin, g)
        X[:, tg, :] = np.where(locked, np.nan, nx)
        Y[:, tg, :] = np.where(locked, np.nan, ny)
        hit = locked.any(axis=1)
        if hit.any():
            t_here = np.where(hit, locked.argmax(axis=1), T)
            earlier = t_here < first_t
            first_t[earlier] = t_here[earlier]
            first_joint[earlier] = tg
    out = {"X": X, "Y": Y, "first_t": first_t, "first_joint": first_joint}
    if with_margin:
        tt = np.arange(T)[None, :]
        gm = np.where(tt <= first_t[:, None], gmin, np.inf)
        out["margin"] = gm.min(axis=1)
    return out


def simulate_scalar(pos0: np.ndarray, steps, fixed, T: int = 200):
    """Scalar per-angle replay of one mechanism (solver.py:142-169, with
    dyad_solve solver.py:123-139): plain Python over t and the plan steps,
    cos/sin/hypot from numpy like the reference.  Returns ("lock", t, joint)
    or ("ok", (n, T, 2) float64)."""
    import math

    pos0 = np.asarray(pos0, dtype=np.float64)
    n = pos0.shape[0]
    p0x, p0y = float(pos0[0, 0]), float(pos0[0, 1])
    r1 = float(np.hypot(pos0[1, 0] - p0x, pos0[1, 1] - p0y))
    if steps:
        R_a, R_b, BR = step_geometry(pos0[None], steps)
        R_a, R_b, BR = R_a[0], R_b[0], BR[0]
    out = np.empty((n, T, 2), dtype=np.float64)
    cur = [(float(x), float(y)) for x, y in pos0]
    cos_t, sin_t = crank_angles(T)
    for t in range(T):
        cur[1] = (p0x + r1 * cos_t[t], p0y + r1 * sin_t[t])
        for s, (tg, a, b) in enumerate(steps):
            pa, pb = cur[a], cur[b]
            dx = pb[0] - pa[0]
            dy = pb[1] - pa[1]
            d = float(np.hypot(dx, dy))
            ra, rb, br = float(R_a[s]), float(R_b[s]), float(BR[s])
            if d < LOCK_EPS or d > ra + rb + LOCK_EPS or d < abs(ra - rb) - LOCK_EPS:
                return ("lock", t, tg)
            x = (d * d + ra * ra - rb * rb) / (2.0 * d)
            h = math.sqrt(max(ra * ra - x * x, 0.0))
            ux, uy = dx / d, dy / d
            cur[tg] = (pa[0] + x * ux - br * h * uy, pa[1] + x * uy + br * h * ux)
        for k in range(n):
            out[k, t, 0] = cur[k][0]
            out[k, t, 1] = cur[k][1]
    return ("ok", out)


def gate(pos0: np.ndarray, steps, fixed, T_low: int = 50, T_high: int = 200):
    """Two-fidelity gate of one topology group (find_valid_variant's
    pattern, generator.py:263-275, with the survivors confirmed as one batch
    as SURVEY.md §8d C3 prescribes): T_low sweep of every candidate, T_high
    only for the T_low survivors.  Returns (valid (B,) bool, low_t (B,)
    int64: the T_low lock step, -1 for T_low survivors)."""
    lo = simulate(pos0, steps, fixed, T_low)
    valid = np.zeros(len(pos0), dtype=bool)
    low_t = np.where(lo["first_t"] < T_low, lo["first_t"], -1)
    surv = np.flatnonzero(lo["first_t"] == T_low)
    if len(surv):
        hi = simulate(np.asarray(pos0)[surv], steps, fixed, T_high)
        valid[surv] = hi["first_t"] == T_high
    return valid, low_t


def trajectories(res) -> np.ndarray:
    """(B, n, T, 2) view of a simulate() result, like the reference's P."""
    return np.stack([res["X"], res["Y"]], axis=-1)


# ---------------------------------------------------------------- curves
def farthest_pair(pts: np.ndarray):
    """Exact O(T^2) search, lexicographically smallest pair on ties
    (curves.py:22-30)."""
    diff = pts[:, None, :] - pts[None, :, :]
    D = np.sqrt((diff * diff).sum(axis=-1))
    i, j = divmod(int(np.argmax(D)), pts.shape[0])
    if i > j:
        i, j = j, i
    return i, j, float(D[i, j])


def _box_center(p: np.ndarray) -> np.ndarray:
    # curves.py:33-36
    return p - (p.min(axis=0) + p.max(axis=0)) / 2.0 + np.array([0.5, 0.5])


def _angle_about_center(p: np.ndarray) -> float:
    # curves.py:39-42
    v = p[0] - np.array([0.5, 0.5])
    a = float(np.arctan2(v[1], v[0]))
    return a if a >= 0.0 else a + 2.0 * np.pi


def normalize(path: np.ndarray) -> np.ndarray:
    """Farthest-pair frame, unit diameter, bbox centred at (0.5, 0.5), and the
    half-turn choice by first-point angle then y-mass (curves.py:45-71)."""
    p = np.asarray(path, dtype=np.float64)
    if p.ndim != 2 or p.shape[1] != 2 or p.shape[0] < 2:
        raise ValueError("path must be a (T, 2) array with T >= 2")
    i, j, d = farthest_pair(p)
    if d <= 0.0:
        raise ValueError("degenerate path: all points coincide")
    v = p[j] - p[i]
    c, s = v[0] / d, v[1] / d
    rot = np.array([[c, s], [-s, c]])
    base = (p - p[i]) @ rot.T / d
    A = _box_center(base)
    Bc = _box_center(-base)
    aa, ab = _angle_about_center(A), _angle_about_center(Bc)
    if abs(aa - ab) <= 1e-12:
        ma = float(np.maximum(A[:, 1] - 0.5, 0.0).sum())
        mb = float(np.maximum(Bc[:, 1] - 0.5, 0.0).sum())
        return A if ma >= mb else Bc
    return A if aa < ab else Bc


def is_normalized(path: np.ndarray, tol: float = NORM_TOL) -> bool:
    """curves.py:74-84."""
    p = np.asarray(path, dtype=np.float64)
    if p.ndim != 2 or p.shape[1] != 2 or p.shape[0] < 2:
        return False
    i, j, d = farthest_pair(p)
    if abs(d - 1.0) > tol or abs(p[i, 1] - p[j, 1]) > tol:
        return False
    mid = (p.min(axis=0) + p.max(axis=0)) / 2.0
    return bool(np.all(np.abs(mid - 0.5) <= tol))


def is_circle(npath: np.ndarray) -> bool:
    """Population variance of radius about (0.5, 0.5), strict < 5e-4
    (curves.py:95-101)."""
    p = np.asarray(npath, dtype=np.float64)
    r = np.hypot(p[:, 0] - 0.5, p[:, 1] - 0.5)
    return bool(np.var(r) < CIRCLE_VARIANCE_THRESHOLD)


def circle_variance(npath: np.ndarray) -> float:
    p = np.asarray(npath, dtype=np.float64)
    return float(np.var(np.hypot(p[:, 0] - 0.5, p[:, 1] - 0.5)))


def frame_stability(path: np.ndarray, rel: float = 1e-6, y_tol: float = 1e-6) -> bool:
    """SURVEY.md §8a parity predicate for normalised curves: the farthest pair
    is unique within relative ``rel`` (the reference's own predicate at 1e-7,
    test_acceptance.py:252-255, loosened for fp32 inputs) and the first point
    of the normalised curve is not within ``y_tol`` of the half-turn boundary
    y = 0.5 (the flip rule, curves.py:63-71)."""
    p = np.asarray(path, dtype=np.float64)
    diff = p[:, None, :] - p[None, :, :]
    D = np.sqrt((diff * diff).sum(axis=-1))
    near = int((D > D.max() * (1.0 - rel)).sum())
    if near != 2:
        return False
    out = normalize(p)
    return abs(out[0, 1] - 0.5) >= y_tol


def chamfer(A: np.ndarray, B: np.ndarray) -> float:
    """Bi-directional mean nearest-neighbour distance (curves.py:123-129)."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    diff = A[:, None, :] - B[None, :, :]
    D = np.sqrt((diff * diff).sum(axis=-1))
    return float(D.min(axis=1).mean() + D.min(axis=0).mean())


def chamfer_direct_block(points: np.ndarray, query: np.ndarray) -> np.ndarray:
    """Direct-difference chamfer of every curve in (C, P, 2) against one
    (Q, 2) query; the cdist form of curves.py:123-129 applied per curve."""
    pts = np.asarray(points, dtype=np.float64)
    q = np.asarray(query, dtype=np.float64)
    out = np.empty(pts.shape[0])
    for c0 in range(0, pts.shape[0], 256):
        blk = pts[c0:c0 + 256]
        dx = blk[:, :, None, 0] - q[None, None, :, 0]
        dy = blk[:, :, None, 1] - q[None, None, :, 1]
        D = np.sqrt(dx * dx + dy * dy)
        out[c0:c0 + 256] = D.min(axis=2).mean(axis=1) + D.min(axis=1).mean(axis=1)
    return out


def chamfer_expansion_block(points: np.ndarray, query: np.ndarray) -> np.ndarray:
    """The atlas scan's expansion-GEMM chamfer (atlas.py:45-55)."""
    C, P, _ = points.shape
    flat = points.reshape(C * P, 2)
    sq = (flat ** 2).sum(axis=1)[:, None] + (query ** 2).sum(axis=1)[None, :] - 2.0 * flat @ query.T
    D = np.sqrt(np.clip(sq, 0.0, None)).reshape(C, P, -1)
    return D.min(axis=2).mean(axis=1) + D.min(axis=1).mean(axis=1)


def resample(path: np.ndarray, count: int) -> np.ndarray:
    """curves.py:164-170."""
    p = np.asarray(path, dtype=np.float64)
    if p.shape[0] <= count:
        return p
    idx = np.linspace(0, p.shape[0] - 1, count).round().astype(np.intp)
    return p[idx]


# ---------------------------------------------------------------- atlas scan
SCAN_CHUNK = 4096  # atlas.py:32


def retrieve(points: np.ndarray, order: np.ndarray, query: np.ndarray, k: int,
             threshold: float, dist_fn=chamfer_expansion_block):
    """Shuffle-and-scan (atlas.py:179-236) over a resident (N, P, 2) store.

    Returns a list of (distance, record index, above_threshold) sorted by
    distance exactly as the reference orders its hits.  ``query`` must already
    be normalised.  The exact-duplicate index of atlas.py:76-80 is restated as
    a byte comparison.
    """
    query = np.asarray(query, dtype=np.float64)
    qb = np.ascontiguousarray(query).tobytes()
    self_idx = None
    if points.shape[1:] == query.shape:
        for i in range(points.shape[0]):
            if points[i].tobytes() == qb:
                self_idx = i  # the dict keeps the LAST duplicate
    hits = []
    if self_idx is not None:
        hits.append((0.0, self_idx))
    seen_d, seen_i = [], []
    for c0 in range(0, len(order), SCAN_CHUNK):
        idx = order[c0:c0 + SCAN_CHUNK]
        dists = dist_fn(points[idx], query)
        for pos in np.nonzero(dists < threshold)[0]:
            if int(idx[pos]) == self_idx:
                continue
            hits.append((float(dists[pos]), int(idx[pos])))
            if len(hits) >= k:
                break
        if len(hits) >= k:
            break
        top = np.argsort(dists, kind="stable")[:k]
        seen_d.append(dists[top])
        seen_i.append(idx[top])
    res = [(d, i, d >= threshold) for d, i in hits]
    if len(res) < k and seen_d:
        all_d = np.concatenate(seen_d)
        all_i = np.concatenate(seen_i)
        used = {i for _, i, _ in res}
        for pos in np.argsort(all_d, kind="stable"):
            if len(res) >= k:
                break
            i = int(all_i[pos])
            if i in used:
                continue
            used.add(i)
            res.append((float(all_d[pos]), i, True))
    res.sort(key=lambda r: r[0])
    return res


def topk_exhaustive(dists: np.ndarray, scan_pos: np.ndarray, k: int):
    """Top-k record indices by (distance, scan position) — the exhaustive
    ordering of test_atlas.py:106-118 / SURVEY.md §8a a-10."""
    key = np.lexsort((scan_pos, dists))
    return key[:k]


def merge_shard_lists(parts: list, k: int) -> dict:
    """Merge of per-shard retrieval lists (numpy dicts of (NQ, k) arrays with
    global ids / scan positions; id < 0 = empty): the scan-order rules of
    atlas.py:207-235 applied to the union of the shards -- non-hits by
    (d, scan position), hits by scan position, hit counts summed."""
    NQ = parts[0]["top_d"].shape[0]
    out = {"top_d": np.full((NQ, k), np.inf, np.float32), "hit_d": np.full((NQ, k), np.inf, np.float32)}
    for n in ("top_id", "top_pos", "hit_id", "hit_pos"):
        out[n] = np.full((NQ, k), -1, np.int64)
    out["n_hits"] = sum(np.asarray(p["n_hits"], np.int64) for p in parts)
    for q in range(NQ):
        for kind in ("top", "hit"):
            d = np.concatenate([np.asarray(p[f"{kind}_d"][q]) for p in parts])
            ids = np.concatenate([np.asarray(p[f"{kind}_id"][q]) for p in parts])
            pos = np.concatenate([np.asarray(p[f"{kind}_pos"][q]) for p in parts])
            keep = ids >= 0
            d, ids, pos = d[keep], ids[keep], pos[keep]
            sel = (np.argsort(pos, kind="stable") if kind == "hit" else np.lexsort((pos, d)))[:k]
            out[f"{kind}_d"][q, :len(sel)] = d[sel]
            out[f"{kind}_id"][q, :len(sel)] = ids[sel]
            out[f"{kind}_pos"][q, :len(sel)] = pos[sel]
    return out


# ---------------------------------------------------------------- coarse filter
def coarse_descriptor(path: np.ndarray) -> np.ndarray:
    """Radial-histogram + extent descriptor (atlas.py:167-172)."""
    path = np.asarray(path, dtype=np.float64)
    r = np.hypot(path[:, 0] - 0.5, path[:, 1] - 0.5)
    hist, _ = np.histogram(r, bins=16, range=(0.0, 0.75))
    hist = hist / max(len(r), 1)
    extent = path.max(axis=0) - path.min(axis=0)
    return np.concatenate([hist, extent])


def coarse_filter(descriptors: np.ndarray, order: np.ndarray, qdesc: np.ndarray, budget: int) -> np.ndarray:
    """Heuristic prefilter (atlas.py:153-166): the ``budget`` records with
    the smallest descriptor L1 distance (stable argsort -> ties by index),
    in scan order."""
    if budget >= len(descriptors):
        return order
    dist = np.abs(descriptors - qdesc[None, :]).sum(axis=1)
    keep = np.argsort(dist, kind="stable")[:budget]
    mask = np.zeros(len(descriptors), dtype=bool)
    mask[keep] = True
    return order[mask[order]]


def curation_keep(mech_id: int, joint_id: int, flagged: bool, keep_rate: float, seed: int) -> bool:
    """Record-keyed keep rule (curves.py:104-110)."""
    if not flagged:
        return True
    return bool(np.random.default_rng([seed, mech_id, joint_id]).random() < keep_rate)
