"""Drop-in curve API backed by the sm_100a normalise / chamfer kernels.

Reference: linkatlas curves.py.  ``normalize`` (curves.py:45-71),
``is_normalized`` (74-84), ``is_circle`` (95-101) and ``chamfer``
(123-129) keep their signatures and errors; their numpy/scipy bodies are
replaced by ``la_normalize`` / ``la_circle_stats`` / ``la_chamfer_topk``.
Topology helpers (``is_arc``, ``plan_ancestry``, ``reduce_mechanism``),
index resampling and the record-keyed curation rule stay host code.

Batch entry points (``normalize_tensors``, ``chamfer_block``) work on
device tensors.
"""

from __future__ import annotations

import numpy as np

from paper_2208_14567_b200 import _native as N
from paper_2208_14567_b200.mechanism import JointType, Mechanism
from paper_2208_14567_b200.solver import SolutionPlan

BOX_CENTER = np.array([0.5, 0.5])
CIRCLE_VARIANCE_THRESHOLD = 5e-4
NORM_TOL = 1e-9


class DegeneratePathError(ValueError):
    """All path points coincide (curves.py:18)."""


# ------------------------------------------------------------ device batch
def normalize_tensors(paths, *, src_row=None, M: int | None = None, out_f64: bool | None = None,
                      rel_tol: float = 1e-6, y_tol: float = 1e-6, want_bbox: bool = False,
                      stream=None) -> dict:
    """la_normalize over device paths.

    paths: (rows, P, 2) float32/float64 CUDA tensor; src_row: optional (M,)
    int64 row indices (gather, e.g. moving-joint rows of a trajectory
    buffer).  Returns dict with ``out`` (M, P, 2), ``pair`` (M, 2) int32,
    ``diameter``, ``is_circle``, ``circle_var``, ``unstable``, ``status``.
    """
    torch = N.require_cuda()
    lib = N.load()
    if paths.dim() != 3 or paths.shape[2] != 2 or not paths.is_cuda:
        raise ValueError("paths must be a (rows, P, 2) CUDA tensor")
    if paths.dtype not in (torch.float32, torch.float64):
        raise ValueError("paths must be float32 or float64")
    paths = paths.contiguous()
    P = paths.shape[1]
    if P < 2:
        raise ValueError("path must be a (T, 2) array with T >= 2")
    if src_row is not None:
        src_row = src_row.to(device=paths.device, dtype=torch.int64).contiguous()
        M = src_row.numel()
    elif M is None:
        M = paths.shape[0]
    in_f64 = paths.dtype == torch.float64
    of64 = in_f64 if out_f64 is None else out_f64
    dev = paths.device
    out = {
        "out": torch.empty((M, P, 2), dtype=torch.float64 if of64 else torch.float32, device=dev),
        "pair": torch.empty((M, 2), dtype=torch.int32, device=dev),
        "diameter": torch.empty(M, dtype=torch.float64, device=dev),
        "is_circle": torch.empty(M, dtype=torch.uint8, device=dev),
        "circle_var": torch.empty(M, dtype=torch.float64, device=dev),
        "unstable": torch.empty(M, dtype=torch.uint8, device=dev),
        "status": torch.empty(M, dtype=torch.int32, device=dev),
    }
    if want_bbox:
        out["bbox"] = torch.empty((M, 4), dtype=torch.float64, device=dev)
    a = N.LaNormArgs()
    a.paths = paths.data_ptr()
    a.in_f64 = int(in_f64)
    a.src_row = N.ptr(src_row)
    a.M, a.P = M, P
    a.out = out["out"].data_ptr()
    a.out_f64 = int(of64)
    a.pair = out["pair"].data_ptr()
    a.diameter = out["diameter"].data_ptr()
    a.is_circle = out["is_circle"].data_ptr()
    a.circle_var = out["circle_var"].data_ptr()
    a.unstable = out["unstable"].data_ptr()
    a.status = out["status"].data_ptr()
    a.bbox = N.ptr(out.get("bbox"))
    a.rel_tol, a.y_tol = rel_tol, y_tol
    N.check(lib.la_normalize(a, N.stream_ptr(stream)), "la_normalize")
    return out


def _as_device_path(path):
    torch = N.require_cuda()
    pts = np.asarray(path, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 2 or pts.shape[0] < 2:
        raise ValueError("path must be a (T, 2) array with T >= 2")
    return torch.from_numpy(np.ascontiguousarray(pts)).cuda()[None]


# ------------------------------------------------------------ drop-in API
def normalize(path: np.ndarray) -> np.ndarray:
    """Unit-diameter, farthest-pair-horizontal, box-centred canonical path
    (curves.py:45-71), computed by la_normalize in f64."""
    res = normalize_tensors(_as_device_path(path), out_f64=True)
    if int(res["status"][0].item()) != 0:
        raise DegeneratePathError("all path points coincident")
    return res["out"][0].cpu().numpy()


def is_normalized(path: np.ndarray, tol: float = NORM_TOL) -> bool:
    """curves.py:74-84: unit diameter, horizontal diameter, centred box."""
    pts = np.asarray(path, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 2 or pts.shape[0] < 2:
        return False
    res = normalize_tensors(_as_device_path(pts), out_f64=True, want_bbox=True)
    if int(res["status"][0].item()) != 0:
        return False
    d = float(res["diameter"][0].item())
    i, j = (int(v) for v in res["pair"][0].tolist())
    if abs(d - 1.0) > tol or abs(pts[i, 1] - pts[j, 1]) > tol:
        return False
    lo_x, lo_y, hi_x, hi_y = res["bbox"][0].tolist()
    center = np.array([(lo_x + hi_x) / 2.0, (lo_y + hi_y) / 2.0])
    return bool(np.all(np.abs(center - BOX_CENTER) <= tol))


def circle_stats(paths, stream=None):
    """(variance, flag) of the is_circle statistic for device paths."""
    torch = N.require_cuda()
    lib = N.load()
    paths = paths.contiguous()
    M, P = paths.shape[0], paths.shape[1]
    var = torch.empty(M, dtype=torch.float64, device=paths.device)
    flag = torch.empty(M, dtype=torch.uint8, device=paths.device)
    N.check(lib.la_circle_stats(paths.data_ptr(), int(paths.dtype == torch.float64), M, P, var.data_ptr(),
                                flag.data_ptr(), N.stream_ptr(stream)), "la_circle_stats")
    return var, flag


def is_circle(npath: np.ndarray) -> bool:
    """Radius variance about (0.5, 0.5) strictly below 5e-4 (curves.py:95-101)."""
    torch = N.require_cuda()
    pts = np.ascontiguousarray(np.asarray(npath, dtype=np.float64))
    _, flag = circle_stats(torch.from_numpy(pts).cuda()[None])
    return bool(int(flag[0].item()))


def chamfer_block(points, query, *, stream=None):
    """Chamfer distance of every curve of a (C, P, 2) block to one (Q, 2)
    query (atlas.py:45-55) — device tensors in, (C,) float32 out."""
    torch = N.require_cuda()
    from paper_2208_14567_b200.atlas import chamfer_scan

    pts = points.to(dtype=torch.float32).contiguous()
    q = query.to(device=pts.device, dtype=torch.float32).contiguous()[None]
    res = chamfer_scan(pts, q, k=0, dense=True, stream=stream)
    return res["all_d"][0]


def chamfer(A: np.ndarray, B: np.ndarray) -> float:
    """Bi-directional mean nearest-neighbour distance (curves.py:123-129)."""
    torch = N.require_cuda()
    a = torch.from_numpy(np.ascontiguousarray(np.asarray(A, dtype=np.float64))).cuda()
    b = torch.from_numpy(np.ascontiguousarray(np.asarray(B, dtype=np.float64))).cuda()
    return float(chamfer_block(a[None], b)[0].item())


# ------------------------------------------------------------ host helpers
def is_arc(mech: Mechanism, joint: int) -> bool:
    """A joint pinned to a fixed neighbour traces an arc (curves.py:87-92)."""
    if not (0 <= joint < mech.n):
        raise IndexError(f"joint {joint} out of range")
    return bool(np.any(mech.types[mech.neighbors(joint)] == JointType.FIXED))


def curation_keep(mech_id: int, joint_id: int, flagged: bool, keep_rate: float, seed: int) -> bool:
    """Record-keyed keep decision (curves.py:104-110)."""
    if not flagged:
        return True
    return bool(np.random.default_rng([seed, mech_id, joint_id]).random() < keep_rate)


def curate(records, keep_rate: float = 0.005, seed: int = 0):
    """Drop 1 - keep_rate of the arc-or-circle records (curves.py:113-120)."""
    for rec in records:
        if curation_keep(rec.mech_id, rec.joint_id, bool(rec.is_arc or rec.is_circle), keep_rate, seed):
            yield rec


def plan_ancestry(plan: SolutionPlan, joint: int) -> set[int]:
    """Joints the plan needs to place ``joint`` (curves.py:132-150)."""
    parents = {s.target: (s.a, s.b) for s in plan.steps}
    if joint not in plan.coverage:
        raise ValueError(f"joint {joint} not covered by plan")
    seen: set[int] = set()
    stack = [joint]
    while stack:
        k = stack.pop()
        if k in seen:
            continue
        seen.add(k)
        if k in parents:
            stack.extend(parents[k])
        elif k == 1:
            stack.append(0)
    seen.update({0, 1})
    return seen


def reduce_mechanism(mech: Mechanism, plan: SolutionPlan, joint: int) -> Mechanism:
    """Sub-mechanism induced by the ancestry of ``joint`` (curves.py:153-161)."""
    keep = np.array(sorted(plan_ancestry(plan, joint)), dtype=np.intp)
    return Mechanism(mech.adjacency[np.ix_(keep, keep)], mech.types[keep], mech.positions0[keep])


def resample(path: np.ndarray, count: int) -> np.ndarray:
    """Index-subsample to ``count`` of the path's own points (curves.py:164-170)."""
    pts = np.asarray(path, dtype=np.float64)
    if pts.shape[0] <= count:
        return pts
    idx = np.linspace(0, pts.shape[0] - 1, count).round().astype(np.intp)
    return pts[idx]
