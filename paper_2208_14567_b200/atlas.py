"""Drop-in numerical atlas: seeded shuffle-and-scan chamfer retrieval on the GPU.

Reference: linkatlas atlas.py.  ``Atlas.retrieve`` (atlas.py:179-252) keeps
its signature and result semantics — hits are the first ``k`` records in the
persisted shuffle order with chamfer distance below ``threshold`` (an exact
duplicate of the query is inserted first at distance 0.0, atlas.py:204-214);
if fewer than ``k`` exist the list is padded with the best remaining records
by (distance, scan position) and flagged ``above_threshold``
(atlas.py:219-235); the result is sorted by distance (atlas.py:236).

The scan itself (``_chamfer_block`` over 4096-record chunks, atlas.py:45-55,
207-222) is one ``la_chamfer_topk`` launch over the device-resident store:
per-warp top-k / first-k-hit lists merged on device.  The exact-duplicate
index of atlas.py:76-80 (a dict of every curve's bytes, infeasible at 10M
records) is replaced by a sorted 64-bit content hash with byte verification.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np
from typing import NamedTuple

from paper_2208_14567_b200 import _native as N
from paper_2208_14567_b200.curves import is_normalized, normalize, normalize_tensors, reduce_mechanism, resample
from paper_2208_14567_b200.mechanism import Mechanism
from paper_2208_14567_b200.solver import compile_plan

logger = logging.getLogger(__name__)

DEFAULT_THRESHOLD = 0.03   # atlas.py:30
DEFAULT_K = 3              # atlas.py:31


from paper_2208_14567_b200.records import FormatError  # noqa: E402  (records.py:26; Atlas.build raises it)


@dataclass
class RetrievalHit:
    mech_id: int
    joint_id: int
    curve: np.ndarray
    distance: float
    mechanism: Mechanism
    above_threshold: bool


# ------------------------------------------------------------ device scan
def chamfer_scan(db, queries, *, k: int = 10, threshold: float = 0.0, order=None, pos_begin: int = 0,
                 pos_end: int | None = None, id_base: int = 0, pos_base: int = 0, pos_map=None,
                 exclude_id: int = -1, dense: bool = False, all_d=None, expansion: bool = False,
                 fix_tol: float = 5e-5, scalar_pipe: bool = False, tensor: bool = False, prune: bool = True,
                 seed_scan: bool = False, multi_query: bool = True, mq_fine: bool = False,
                 cells=None, index_mq: bool = False, stream=None) -> dict:
    """One la_chamfer_topk launch.

    ``cells`` (``chamfer_index(db)``; single-query pruned scans): every curve
    is first bounded from its index rows -- the row term from its 2-byte
    cells, the column term from its coarse distance bytes -- against the k-th
    best of a seed scan over a 1/64 prefix, and only the survivors' points
    are streamed; the lists are identical to the scan without it
    (``n_stage[0]`` / ``[1]`` count the survivors of its two levels).
    ``index_mq`` uses the index for several queries too (a multi-query bound
    step, per-query survivor scans: faster than the multi-query kernel for
    few queries on a large database, slower for many on a small one; off).

    ``prune`` (top-k scans of >= 65,536 positions without dense output):
    curves whose lower bound (query distance grid, first chamfer term)
    exceeds the running k-th best are skipped; the lists are identical to
    the unpruned scan (``prune=False``: every curve evaluated).
    ``seed_scan``: seed the pruning bound with an exact scan of a 1/128
    prefix first (off by default; measured slower than the slot minima).
    ``multi_query`` (pruned scans with several queries): groups of queries
    share each streamed curve and a stage-0 bound on a grid common to the
    group (``mq_fine``: 64x64 instead of 32x32); ``n_stage`` (5,) counts the
    (query, curve) pairs surviving its five bound stages.

    db: (N, P, 2) float32 CUDA tensor; queries: (NQ, Q, 2) float32.  order:
    optional (N,) int64 device tensor, record index at each scan position.
    Returns ``top_d``/``top_id``/``top_pos`` (NQ, k): best non-hits by
    (d, pos); ``hit_d``/``hit_id``/``hit_pos``: first k hits (d < threshold)
    by pos; ``n_hits`` (NQ,); ``all_d`` (NQ, N) when ``dense``.
    Missing entries have id -1 and d = inf.  ``expansion`` selects the
    |a|^2+|q|^2-2a.q inner loop (FFMA2) with a per-curve rigorous rounding
    bound; curves whose bound exceeds ``fix_tol`` are recomputed with direct
    differences, so every distance is within fix_tol of the exact fp32-input
    value.
    """
    torch = N.require_cuda()
    lib = N.load()
    if db.dtype != torch.float32 or db.dim() != 3 or db.shape[2] != 2 or not db.is_cuda:
        raise ValueError("db must be a (N, P, 2) float32 CUDA tensor")
    if queries.dim() == 2:
        queries = queries[None]
    queries = queries.to(device=db.device, dtype=torch.float32).contiguous()
    db = db.contiguous()
    Nn, P = db.shape[0], db.shape[1]
    NQ, Q = queries.shape[0], queries.shape[1]
    if k > N.LA_MAX_TOPK:
        raise ValueError(f"k <= {N.LA_MAX_TOPK} supported")
    pe = Nn if pos_end is None else int(pos_end)
    dev = db.device
    out: dict = {}
    kk = max(int(k), 0)
    if kk > 0:
        for name, dt in (("top_d", torch.float32), ("top_id", torch.int64), ("top_pos", torch.int64),
                         ("hit_d", torch.float32), ("hit_id", torch.int64), ("hit_pos", torch.int64)):
            out[name] = torch.empty((NQ, kk), dtype=dt, device=dev)
    out["n_hits"] = torch.zeros(NQ, dtype=torch.int64, device=dev)
    out["n_full"] = torch.zeros(NQ, dtype=torch.int64, device=dev)  # curves evaluated in full (fast path)
    out["n_stage"] = torch.zeros(5, dtype=torch.int64, device=dev)
    if dense and all_d is None:
        all_d = torch.full((NQ, Nn), float("nan"), dtype=torch.float32, device=dev)
    if all_d is not None:
        out["all_d"] = all_d
    if order is not None:
        order = order.to(device=dev, dtype=torch.int64).contiguous()
    if pos_map is not None:
        pos_map = pos_map.to(device=dev, dtype=torch.int64).contiguous()
    a = N.LaChamferArgs()
    a.db, a.N, a.P = db.data_ptr(), Nn, P
    a.queries, a.NQ, a.Q = queries.data_ptr(), NQ, Q
    a.order = N.ptr(order)
    a.pos_begin, a.pos_end = int(pos_begin), pe
    a.id_base, a.pos_base = int(id_base), int(pos_base)
    a.pos_map = N.ptr(pos_map)
    a.k = kk
    a.threshold = float(threshold) if np.isfinite(threshold) else (3.0e38 if threshold > 0 else -3.0e38)
    a.exclude_id = int(exclude_id)
    for name in ("top_d", "top_id", "top_pos", "hit_d", "hit_id", "hit_pos"):
        setattr(a, name, N.ptr(out.get(name)))
    a.n_hits = out["n_hits"].data_ptr()
    a.all_d = N.ptr(all_d)
    a.flags = ((N.LA_CH_EXPANSION if expansion else 0) | (N.LA_CH_SCALAR_PIPE if scalar_pipe else 0)
               | (N.LA_CH_TENSOR if tensor else 0) | (0 if prune else N.LA_CH_NO_PRUNE)
               | (N.LA_CH_SEED_SCAN if seed_scan else 0) | (0 if multi_query else N.LA_CH_NO_MQ)
               | (N.LA_CH_MQ_FINE if mq_fine else 0) | (N.LA_CH_INDEX_MQ if index_mq else 0))
    a.fixup_below = float(fix_tol)
    a.n_full = out["n_full"].data_ptr()
    a.n_stage = out["n_stage"].data_ptr()
    coarse = fine = None
    if isinstance(cells, ChamferIndex):
        cells, coarse, fine = cells.cells, cells.coarse, cells.fine
    if cells is not None:
        if cells.dtype != torch.uint16 or tuple(cells.shape) != (Nn, (P + 15) & ~15) or not cells.is_cuda:
            raise ValueError("cells must be chamfer_index(db) (or its (N, P rounded up to 16) uint16 cells)")
        cells = cells.contiguous()
        if coarse is not None and (coarse.dtype != torch.uint8 or tuple(coarse.shape) != (Nn, 256)):
            raise ValueError("coarse must be the (N, 256) uint8 tensor of chamfer_index(db)")
        if fine is not None and (fine.dtype != torch.uint8 or tuple(fine.shape) != (Nn, 1024)):
            raise ValueError("fine must be the (N, 1024) uint8 tensor of chamfer_index(db)")
    a.cells = N.ptr(cells)
    a.coarse = N.ptr(coarse.contiguous() if coarse is not None else None)
    a.fine = N.ptr(fine.contiguous() if (fine is not None and coarse is not None) else None)
    wsb = int(lib.la_chamfer_workspace(a))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    a.ws, a.ws_bytes = ws.data_ptr(), wsb
    N.check(lib.la_chamfer_topk(a, N.stream_ptr(stream)), "la_chamfer_topk")
    out["_ws"] = ws  # keep alive until the stream consumes it
    return out


class ChamferIndex(NamedTuple):
    """la_chamfer_index outputs for one database: ``cells`` (N, P rounded up
    to 16) uint16, ``coarse`` (N, 256) uint8 (or None) and ``fine`` (N, 1024)
    uint8 (or None)."""
    cells: object
    coarse: object
    fine: object = None


def chamfer_index(db, coarse: bool = True, fine: bool = True, stream=None) -> ChamferIndex:
    """Index of a curve database (la_chamfer_index): the 64 x 64 grid cell of
    every point (2 bytes; row padding: the null cell); with ``coarse``, each
    curve's 16 x 16 distance table (256 bytes, the bound step's column term);
    with ``fine``, its 32 x 32 table (1 KB, read for the bound step's
    survivors only).  Pass it to ``chamfer_scan(cells=...)``."""
    torch = N.require_cuda()
    lib = N.load()
    if db.dtype != torch.float32 or db.dim() != 3 or db.shape[2] != 2 or not db.is_cuda:
        raise ValueError("db must be a (N, P, 2) float32 CUDA tensor")
    db = db.contiguous()
    cells = torch.empty((db.shape[0], (db.shape[1] + 15) & ~15), dtype=torch.uint16, device=db.device)
    cd = torch.empty((db.shape[0], 256), dtype=torch.uint8, device=db.device) if coarse else None
    fd = torch.empty((db.shape[0], 1024), dtype=torch.uint8, device=db.device) if (coarse and fine) else None
    N.check(lib.la_chamfer_index(db.data_ptr(), db.shape[0], db.shape[1], cells.data_ptr(), N.ptr(cd), N.ptr(fd),
                                 N.stream_ptr(stream)), "la_chamfer_index")
    return ChamferIndex(cells, cd, fd)


_EDGES = np.linspace(0.0, 0.75, 17)  # np.histogram(bins=16, range=(0, .75)) edges (atlas.py:169)


def coarse_descriptors(paths) -> "torch.Tensor":
    """Atlas._descriptor (atlas.py:167-172) for a (M, P, 2) float64 CUDA
    tensor -> (M, 18) float64, bit-identical to the reference."""
    torch = N.require_cuda()
    lib = N.load()
    if paths.dtype != torch.float64 or not paths.is_cuda or paths.dim() != 3 or paths.shape[2] != 2:
        raise ValueError("paths must be a (M, P, 2) float64 CUDA tensor")
    paths = paths.contiguous()
    M, P, _ = paths.shape
    desc = torch.empty((M, 18), dtype=torch.float64, device=paths.device)
    N.check(lib.la_coarse_descriptors(paths.data_ptr(), M, P, _EDGES.ctypes.data, desc.data_ptr(), N.stream_ptr()),
            "la_coarse_descriptors")
    return desc


def coarse_select(desc, qdesc, budget: int, order=None, *, return_dist: bool = False):
    """Keep the ``budget`` records nearest ``qdesc`` in descriptor L1
    distance, ties by index (stable argsort, atlas.py:162-166), returned in
    scan order (``order`` filtered; identity when None).  Device int64."""
    torch = N.require_cuda()
    lib = N.load()
    M = desc.shape[0]
    k = int(min(max(budget, 0), M))
    dev = desc.device
    out = torch.empty(k, dtype=torch.int64, device=dev)
    dist = torch.empty(M, dtype=torch.float64, device=dev) if return_dist else None
    if order is not None:
        order = order.to(device=dev, dtype=torch.int64).contiguous()
    ws = torch.empty(max(int(lib.la_coarse_workspace(M)), 1), dtype=torch.uint8, device=dev)
    q = qdesc.to(device=dev, dtype=torch.float64).contiguous().reshape(18)
    N.check(lib.la_coarse_select(desc.contiguous().data_ptr(), M, q.data_ptr(), k, N.ptr(order), out.data_ptr(),
                                 N.ptr(dist), ws.data_ptr(), ws.numel(), N.stream_ptr()), "la_coarse_select")
    return (out, dist) if return_dist else out


def assemble_hits(hit_d, hit_id, top_d, top_id, k, threshold, self_idx=None):
    """Host assembly of the retrieve() result from the device lists.

    Mirrors atlas.py:201-236: self hit first (0.0), scan-order hits up to k,
    padding by (d, pos) flagged above threshold, final stable sort by d.
    Returns [(distance, record, above_threshold)].
    """
    res = []
    if self_idx is not None:
        res.append((0.0, int(self_idx), 0.0 >= threshold))
    for d, i in zip(hit_d, hit_id):
        if len(res) >= k or i < 0:
            break
        res.append((float(d), int(i), False))
    if len(res) < k:
        used = {r[1] for r in res}
        for d, i in zip(top_d, top_id):
            if len(res) >= k:
                break
            if i < 0 or int(i) in used:
                continue
            used.add(int(i))
            res.append((float(d), int(i), True))
    res.sort(key=lambda r: r[0])
    return res


def _content_hash(points: np.ndarray) -> np.ndarray:
    """64-bit multiplicative hash of each record's raw f64 bytes."""
    n = points.shape[0]
    if n == 0:
        return np.zeros(0, dtype=np.uint64)
    words = np.ascontiguousarray(points).reshape(n, -1).view(np.uint64)
    mult = (np.arange(words.shape[1], dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) | np.uint64(1)
    with np.errstate(over="ignore"):
        h = np.zeros(n, dtype=np.uint64)
        for c0 in range(0, words.shape[1], 64):
            h += (words[:, c0:c0 + 64] * mult[c0:c0 + 64]).sum(axis=1, dtype=np.uint64)
    return h


class Atlas:
    """Read-only curve store with a persisted shuffle order (atlas.py:58-80)."""

    def __init__(self, points, mech_ids, joint_ids, mechanisms: dict[int, Mechanism], seed: int):
        self.points = np.asarray(points, dtype=np.float64)
        self.mech_ids = np.asarray(mech_ids, dtype=np.int64)
        self.joint_ids = np.asarray(joint_ids, dtype=np.int64)
        self.mechanisms = mechanisms
        self.seed = int(seed)
        self.order = np.random.default_rng(self.seed).permutation(len(self.points))
        self._descriptors = None
        h = _content_hash(self.points)
        self._hash_order = np.argsort(h, kind="stable")
        self._hash_sorted = h[self._hash_order]
        self._dev = None
        self._order_dev = None

    def __len__(self) -> int:
        return len(self.points)

    @classmethod
    def build(cls, records, mechanisms: dict[int, Mechanism], seed: int = 0,
              resample_to: int | None = None) -> "Atlas":
        """atlas.py:85-110; resampled curves are renormalised in one batch."""
        mech_ids, joint_ids, stack = [], [], []
        for rec in records:
            if rec.mech_id not in mechanisms:
                raise FormatError(f"curve references missing mechanism {rec.mech_id}")
            pts = np.asarray(rec.points, dtype=np.float64)
            if resample_to is not None and pts.shape[0] > resample_to:
                pts = resample(pts, resample_to)
                pts = ("renorm", pts)
            mech_ids.append(rec.mech_id)
            joint_ids.append(rec.joint_id)
            stack.append(pts)
        renorm = [i for i, p in enumerate(stack) if isinstance(p, tuple)]
        if renorm:
            torch = N.require_cuda()
            batch = torch.from_numpy(np.stack([stack[i][1] for i in renorm])).cuda()
            res = normalize_tensors(batch, out_f64=True)
            if bool((res["status"] != 0).any()):
                from paper_2208_14567_b200.curves import DegeneratePathError

                raise DegeneratePathError("all path points coincident")
            outs = res["out"].cpu().numpy()
            for j, i in enumerate(renorm):
                stack[i] = outs[j]
        points = np.zeros((0, 0, 2)) if not stack else np.stack(stack)
        return cls(points, np.array(mech_ids), np.array(joint_ids), mechanisms, seed)

    # -- persistence (atlas.py:114-149) ----------------------------------
    def save(self, directory) -> None:
        """meta.json + curves.ldjson (+ .npz sidecar) + mechanisms.ldjson in
        the reference's record format."""
        import json
        from pathlib import Path

        from paper_2208_14567_b200 import records as R

        d = Path(directory)
        d.mkdir(parents=True, exist_ok=True)
        (d / "meta.json").write_text(json.dumps({"seed": self.seed, "size": len(self)}))
        flags = np.zeros(len(self), dtype=bool)
        R.write_curve_arrays(d / "curves.ldjson", self.mech_ids, self.joint_ids, flags, flags, self.points)
        R.write_curves_npz_arrays(d / "curves.npz", self.mech_ids, self.joint_ids, flags, flags, self.points)
        R.write_records(d / "mechanisms.ldjson", "mechanism",
                        [R.mechanism_to_record(m, mid) for mid, m in sorted(self.mechanisms.items())])

    @classmethod
    def load(cls, directory) -> "Atlas":
        import json
        from pathlib import Path

        from paper_2208_14567_b200 import records as R

        d = Path(directory)
        meta = json.loads((d / "meta.json").read_text())
        npz = d / "curves.npz"
        curves = R.read_curves_npz(npz) if npz.exists() else list(R.RecordReader(d / "curves.ldjson", "curve"))
        mechs = {rec.id: R.record_to_mechanism(rec) for rec in R.RecordReader(d / "mechanisms.ldjson", "mechanism")}
        return cls.build(curves, mechs, seed=meta["seed"])

    # -- device residency ------------------------------------------------
    def device_points(self):
        torch = N.require_cuda()
        if self._dev is None:
            self._dev = torch.from_numpy(self.points.astype(np.float32)).cuda()
        return self._dev

    def device_cells(self):
        """Cell index of the device curves (built once, chamfer_index)."""
        if getattr(self, "_cells_dev", None) is None:
            self._cells_dev = chamfer_index(self.device_points())
        return self._cells_dev

    def exact_index(self, query: np.ndarray) -> int | None:
        """Index of the LAST stored curve byte-identical to ``query``
        (the dict comprehension of atlas.py:78-80 keeps the last)."""
        q = np.ascontiguousarray(np.asarray(query, dtype=np.float64))
        if len(self) == 0 or q.shape != self.points.shape[1:]:
            return None
        h = _content_hash(q[None])[0]
        lo = np.searchsorted(self._hash_sorted, h, side="left")
        hi = np.searchsorted(self._hash_sorted, h, side="right")
        found = None
        qb = q.tobytes()
        for idx in sorted(self._hash_order[lo:hi].tolist()):
            if self.points[idx].tobytes() == qb:
                found = idx
        return found

    # -- coarse prefilter (atlas.py:153-177) on the device -----------------
    def device_descriptors(self, chunk: int = 1 << 18):
        """(N, 18) f64 descriptors, computed once from the f64 curves."""
        torch = N.require_cuda()
        if self._descriptors is None:
            desc = torch.empty((len(self), 18), dtype=torch.float64, device="cuda")
            for c0 in range(0, len(self), chunk):
                c1 = min(len(self), c0 + chunk)
                desc[c0:c1] = coarse_descriptors(torch.from_numpy(self.points[c0:c1]).cuda())
            self._descriptors = desc
        return self._descriptors

    def device_order(self):
        torch = N.require_cuda()
        if self._order_dev is None:
            self._order_dev = torch.from_numpy(np.ascontiguousarray(self.order, dtype=np.int64)).cuda()
        return self._order_dev

    def _coarse_scan(self, query: np.ndarray, budget: int, mode: str):
        """Device scan list (int64 tensor) of coarse_filter."""
        torch = N.require_cuda()
        if mode == "exact" or budget >= len(self):
            return self.device_order()
        q = np.ascontiguousarray(np.asarray(query, dtype=np.float64))
        qd = coarse_descriptors(torch.from_numpy(q[None]).cuda())[0]
        return coarse_select(self.device_descriptors(), qd, int(budget), self.device_order())

    def coarse_filter(self, query: np.ndarray, budget: int, mode: str = "heuristic") -> np.ndarray:
        """Candidate record indices in scan order (atlas.py:153-164)."""
        if mode == "exact" or budget >= len(self):
            return self.order
        return self._coarse_scan(query, budget, mode).cpu().numpy()

    # -- search ----------------------------------------------------------
    def retrieve(self, query: np.ndarray, k: int = DEFAULT_K, threshold: float = DEFAULT_THRESHOLD,
                 budget: int | None = None, filter_mode: str = "exact") -> list[RetrievalHit]:
        """Shuffle-and-scan retrieval (atlas.py:179-252) on the GPU."""
        if len(self) == 0:
            logger.warning("retrieve on an empty atlas")
            return []
        torch = N.require_cuda()
        query = np.asarray(query, dtype=np.float64)
        if not is_normalized(query):
            query = normalize(query)
        scan = self.device_order() if budget is None else self._coarse_scan(query, budget, filter_mode)
        self_idx = self.exact_index(query)
        if not (1 <= k <= N.LA_MAX_TOPK):
            return self._retrieve_large(query, k, threshold, scan.cpu().numpy(), self_idx)
        db = self.device_points()
        res = chamfer_scan(db, torch.from_numpy(query.astype(np.float32)).cuda()[None],
                           k=int(k), threshold=threshold, order=scan,
                           pos_end=int(scan.numel()), exclude_id=-1 if self_idx is None else int(self_idx),
                           cells=self.device_cells() if scan.numel() >= (1 << 16) else None)
        host = {n: res[n][0].cpu().numpy() for n in ("hit_d", "hit_id", "top_d", "top_id")}
        rows = assemble_hits(host["hit_d"], host["hit_id"], host["top_d"], host["top_id"], int(k), threshold,
                             self_idx)
        return [self._hit(d, i, above) for d, i, above in rows]

    def _retrieve_large(self, query, k, threshold, scan, self_idx):
        """k beyond the per-warp list size: dense distances, host ordering."""
        torch = N.require_cuda()
        db = self.device_points()
        res = chamfer_scan(db, torch.from_numpy(query.astype(np.float32)).cuda()[None], k=0, dense=True)
        d = res["all_d"][0].cpu().numpy().astype(np.float64)
        ds = d[scan]
        hits_pos = [p for p in np.flatnonzero(ds < threshold) if scan[p] != self_idx]
        cap = max(int(k), 1) - (1 if self_idx is not None else 0)
        hits_pos = np.array(hits_pos[:max(cap, 0)], dtype=np.int64)
        used = set(int(scan[p]) for p in hits_pos) | ({int(self_idx)} if self_idx is not None else set())
        rest = np.array([p for p in np.lexsort((np.arange(len(ds)), ds)) if int(scan[p]) not in used],
                        dtype=np.int64)
        rows = assemble_hits(ds[hits_pos], scan[hits_pos], ds[rest], scan[rest], int(k), threshold, self_idx)
        return [self._hit(dd, i, above) for dd, i, above in rows]

    def _hit(self, d: float, i: int, above: bool) -> RetrievalHit:
        mech = self.mechanisms[int(self.mech_ids[i])]
        reduced = reduce_mechanism(mech, compile_plan(mech), int(self.joint_ids[i]))
        return RetrievalHit(mech_id=int(self.mech_ids[i]), joint_id=int(self.joint_ids[i]),
                            curve=self.points[i], distance=float(d), mechanism=reduced,
                            above_threshold=bool(above))


def build_atlas(records, mechanisms, seed: int = 0, resample_to: int | None = None) -> Atlas:
    return Atlas.build(records, mechanisms, seed=seed, resample_to=resample_to)
