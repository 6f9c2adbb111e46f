"""Drop-in solver API backed by the sm_100a simulation kernel.

Reference: linkatlas solver.py.  The signatures, result types and error
behaviour of ``compile_plan``, ``plan_geometry``, ``dyad_solve``,
``simulate``, ``simulate_batch`` and ``check_feasible`` are kept; the numpy
bodies (solver.py:105-249) are replaced by ``la_simulate`` /
``la_plan_geometry`` / ``la_dyad_solve`` (include/links_b200.h).  The
topology walk of ``compile_plan`` (solver.py:71-102) stays host code: it is
integer work done once per topology, not per candidate.

Tensor-level entry points (``PlanTable``, ``simulate_tensors``) serve mixed
topologies in one launch and keep results on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2208_14567_b200 import _native as N
from paper_2208_14567_b200.mechanism import JointType, Mechanism

LOCK_EPS = 1e-9                 # solver.py:19 (the kernels hard-code the same)
DEFAULT_FIXUP_TAU = 2e-6  # floor of the error-model margin test (sim.cu solve32)


class PlanError(ValueError):
    """Topology not dyadically solvable or initial pose degenerate (solver.py:22)."""


@dataclass(frozen=True)
class PlanStep:
    target: int
    a: int
    b: int


@dataclass(frozen=True)
class SolutionPlan:
    n: int
    fixed: tuple[int, ...]
    steps: tuple[PlanStep, ...]
    r_a: np.ndarray | None
    r_b: np.ndarray | None
    branch: np.ndarray | None

    @property
    def coverage(self) -> frozenset[int]:
        return frozenset(self.fixed) | {1} | {s.target for s in self.steps}


@dataclass(frozen=True)
class Trajectory:
    positions: np.ndarray  # (n, T, 2)

    @property
    def T(self) -> int:
        return self.positions.shape[1]

    @property
    def n(self) -> int:
        return self.positions.shape[0]


@dataclass(frozen=True)
class Locking:
    step: int
    joint: int


SimOutcome = Trajectory | Locking


# ------------------------------------------------------------ host: topology
def compile_order(adjacency: np.ndarray, types: np.ndarray) -> tuple[tuple[int, ...], tuple[PlanStep, ...]]:
    """The two-known-neighbours walk of solver.py:71-94 on the joint graph.

    Seeds are every Fixed joint plus the crank tip; each pass scans unknown
    joints in ascending order and a joint with >= 2 known neighbours joins
    (with its first two known neighbours) immediately.  Raises PlanError on a
    stall.
    """
    adj = np.asarray(adjacency)
    n = adj.shape[0]
    fixed = tuple(int(k) for k in np.flatnonzero(np.asarray(types) == JointType.FIXED))
    known = np.zeros(n, dtype=bool)
    known[list(fixed)] = True
    if n > 1:
        known[1] = True
    todo = [k for k in range(n) if not known[k]]
    nbrs = [np.flatnonzero(adj[k]) for k in range(n)]
    steps: list[PlanStep] = []
    while todo:
        moved = False
        rest = []
        for k in todo:
            kn = [int(v) for v in nbrs[k] if known[v]]
            if len(kn) >= 2:
                steps.append(PlanStep(k, kn[0], kn[1]))
                known[k] = True
                moved = True
            else:
                rest.append(k)
        if not moved:
            raise PlanError(f"not dyadically solvable: joints {sorted(rest)} unreachable")
        todo = rest
    return fixed, tuple(steps)


def compile_plan(mech: Mechanism) -> SolutionPlan:
    """Solve order + (when the pose is set) its geometry (solver.py:71-102).

    The geometry is computed by ``la_plan_geometry`` on the device.
    """
    fixed, steps = compile_order(mech.adjacency, mech.types)
    bare = SolutionPlan(mech.n, fixed, steps, None, None, None)
    if np.isnan(mech.positions0).any():
        return bare
    r_a, r_b, branch = plan_geometry(bare, mech.positions0)
    if np.any((r_a < LOCK_EPS) | (r_b < LOCK_EPS)):
        raise PlanError("degenerate branch: zero-length bar at initial pose")
    return SolutionPlan(mech.n, fixed, steps, r_a, r_b, branch)


# ------------------------------------------------------------ plan tables
def _pack_plan(plan: SolutionPlan) -> bytes:
    if plan.n > N.LA_MAX_JOINTS:
        raise ValueError(f"mechanisms up to {N.LA_MAX_JOINTS} joints are supported (got {plan.n})")
    if len(plan.steps) > N.LA_MAX_STEPS:
        raise ValueError(f"plans up to {N.LA_MAX_STEPS} dyad steps are supported")
    rec = N.LaPlan()
    rec.n = plan.n
    rec.nsteps = len(plan.steps)
    mask = 0
    for j in plan.fixed:
        mask |= 1 << int(j)
    rec.fixed_mask = mask
    for s, st in enumerate(plan.steps):
        rec.step[s][0], rec.step[s][1], rec.step[s][2] = st.target, st.a, st.b
    return bytes(rec)


@dataclass
class PlanTable:
    """Device-resident array of compiled plans (la_plan records, 64 B each).

    Built from SolutionPlan objects, or from raw records (``from_records``,
    e.g. the native generator's output)."""

    plans: list[SolutionPlan]
    device: object = None
    _dev: object = field(default=None, repr=False)
    _raw: np.ndarray | None = field(default=None, repr=False)
    _ns: np.ndarray | None = field(default=None, repr=False)

    @classmethod
    def from_records(cls, raw: np.ndarray, n: np.ndarray, device=None) -> "PlanTable":
        raw = np.ascontiguousarray(raw, dtype=np.uint8)
        if raw.size % 64:
            raise ValueError("plan records are 64 bytes each")
        return cls([], device=device, _raw=raw, _ns=np.asarray(n, dtype=np.int32))

    @property
    def G(self) -> int:
        return len(self._ns) if self._raw is not None else len(self.plans)

    @property
    def max_n(self) -> int:
        if self._raw is not None:
            return int(self._ns.max())
        return max(p.n for p in self.plans)

    def host_bytes(self) -> np.ndarray:
        if self._raw is not None:
            return self._raw
        return np.frombuffer(b"".join(_pack_plan(p) for p in self.plans), dtype=np.uint8)

    def tensor(self):
        torch = N.require_cuda()
        if self._dev is None:
            dev = self.device if self.device is not None else torch.device("cuda")
            self._dev = torch.from_numpy(self.host_bytes().copy()).to(dev)
        return self._dev


_CRANK: dict = {}


def crank_table(T: int, device=None):
    """cos/sin of theta_t = 2*pi*t/T exactly as solver.py:156-158 computes
    them (numpy f64), interleaved [T][2] on the device (cached)."""
    torch = N.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (int(T), str(dev))
    t = _CRANK.get(key)
    if t is None:
        th = 2.0 * np.pi * np.arange(T) / T
        cs = np.stack([np.cos(th), np.sin(th)], axis=1)
        t = torch.from_numpy(np.ascontiguousarray(cs)).to(dev)
        _CRANK[key] = t
    return t


# ------------------------------------------------------------ device entry
def simulate_tensors(pos0, table: PlanTable, T: int = 200, topo=None, *, write_traj: bool = True,
                     traj=None, traj_stride: int | None = None, traj_row=None, low: bool = False,
                     traj_f64: bool = False, cand=None, cand_count=None,
                     fixup_tau: float = DEFAULT_FIXUP_TAU, fp64: bool = False, gate_only: bool = False,
                     coarse: bool = True, counters=None, stream=None, exact: bool | None = None,
                     _extra_flags: int = 0, _screen: tuple[int, int] = (0, 0),
                     traj2=None, traj_row2=None, _outputs=None) -> dict:
    """Launch la_simulate on device tensors.

    pos0: (B, S, 2) float64 CUDA tensor (S >= every plan's n); topo: (B,)
    int32 plan indices or None (all plan 0).  Returns a dict with
    ``first_t`` / ``first_joint`` (int32, (B,)), ``traj`` ((rows, T, 2)
    float32 — float64 with ``traj_f64`` — when written) and ``low_t`` /
    ``low_joint`` when ``low``.  ``cand`` (int64 device indices, optional
    device count ``cand_count``) gathers the work items; outputs are then
    indexed by work item.  ``exact`` (default: on for f64 paths or the
    all-f64 mode) runs the f64 rounds in numpy's operation order with IEEE
    operations (LA_SIM_EXACT64): f64 paths and the lock decisions of replayed
    lanes are then bit-identical to the reference.
    """
    torch = N.require_cuda()
    lib = N.load()
    if pos0.dtype != torch.float64 or not pos0.is_cuda or pos0.dim() != 3 or pos0.shape[2] != 2:
        raise ValueError("pos0 must be a (B, S, 2) float64 CUDA tensor")
    pos0 = pos0.contiguous()
    B, S, _ = pos0.shape
    if S < table.max_n:
        raise ValueError("pos0 row stride smaller than a plan's joint count")
    dev = pos0.device
    if topo is not None:
        topo = topo.to(device=dev, dtype=torch.int32).contiguous()
    ts = int(traj_stride if traj_stride is not None else table.max_n)
    items = B if cand is None else cand.numel()
    if cand is not None:
        cand = cand.to(device=dev, dtype=torch.int64).contiguous()
    if _outputs is not None:  # caller-provided flag buffers (scatter mode)
        out = {"first_t": _outputs[0], "first_joint": _outputs[1]}
    else:
        out = {
            "first_t": torch.empty(items, dtype=torch.int32, device=dev),
            "first_joint": torch.empty(items, dtype=torch.int32, device=dev),
        }
    if write_traj:
        if traj is None:
            rows = items * ts if traj_row is None else None
            if rows is None:
                raise ValueError("traj_row requires an explicit traj buffer")
            traj = torch.empty((rows, T, 2), dtype=torch.float64 if traj_f64 else torch.float32, device=dev)
        elif traj.dtype != (torch.float64 if traj_f64 else torch.float32):
            raise ValueError("traj dtype does not match traj_f64")
        out["traj"] = traj
    if low:
        out["low_t"] = torch.empty(items, dtype=torch.int32, device=dev)
        out["low_joint"] = torch.empty(items, dtype=torch.int32, device=dev)
    if counters is not None and (counters.numel() < 8 or counters.dtype != torch.int64 or not counters.is_cuda):
        raise ValueError("counters must be an int64 CUDA tensor with >= 8 entries")
    flags = 0
    if write_traj:
        flags |= N.LA_SIM_WRITE_TRAJ
    if fp64:
        flags |= N.LA_SIM_FP64
    if gate_only:
        flags |= N.LA_SIM_GATE_ONLY
    if not coarse:
        flags |= N.LA_SIM_NO_COARSE
    if traj_f64:
        flags |= N.LA_SIM_TRAJ_F64
    if exact if exact is not None else (traj_f64 or fp64):
        flags |= N.LA_SIM_EXACT64
    flags |= int(_extra_flags)
    a = N.LaSimArgs()
    a.pos0 = pos0.data_ptr()
    a.topo = N.ptr(topo)
    a.plans = table.tensor().data_ptr()
    a.crank_cs = crank_table(T, dev).data_ptr()
    a.B, a.G, a.pos_stride, a.T, a.traj_stride = B, table.G, S, T, ts
    a.traj = N.ptr(out.get("traj"))
    a.traj_row = N.ptr(traj_row)
    a.cand = N.ptr(cand)
    a.n_cand = items if cand is not None else 0
    a.cand_count = N.ptr(cand_count)
    a.first_t = out["first_t"].data_ptr()
    a.first_joint = out["first_joint"].data_ptr()
    a.low_t = N.ptr(out.get("low_t"))
    a.low_joint = N.ptr(out.get("low_joint"))
    a.counters = N.ptr(counters)
    a.fixup_tau = float(fixup_tau)
    a.flags = flags
    a.screen_refill, a.screen_replay = int(_screen[0]), int(_screen[1])
    if (traj2 is None) != (traj_row2 is None):
        raise ValueError("traj2 and traj_row2 go together")
    a.traj2, a.traj_row2 = N.ptr(traj2), N.ptr(traj_row2)
    N.check(lib.la_simulate(a, N.stream_ptr(stream)), "la_simulate")
    return out


def compact_valid(first_t, T: int, stream=None):
    """Ascending indices of candidates with first_t == T (la_compact_valid)."""
    torch = N.require_cuda()
    lib = N.load()
    B = first_t.numel()
    idx = torch.empty(max(B, 1), dtype=torch.int64, device=first_t.device)
    cnt = torch.empty(1, dtype=torch.int64, device=first_t.device)  # written by the scan (or zeroed for B == 0)
    wsb = int(lib.la_compact_workspace(B))
    ws = torch.empty(wsb, dtype=torch.uint8, device=first_t.device)
    N.check(lib.la_compact_valid(first_t.data_ptr(), B, T, idx.data_ptr(), cnt.data_ptr(),
                                 ws.data_ptr(), wsb, N.stream_ptr(stream)), "la_compact_valid")
    return idx, cnt


def compact_rows(first_t, T: int, table: "PlanTable", topo=None, stream=None):
    """la_compact_rows: ascending indices of candidates with first_t == T,
    their dense first path rows (running sum of plan joint counts) and, on
    the device, the count and the total number of rows."""
    torch = N.require_cuda()
    lib = N.load()
    B = first_t.numel()
    dev = first_t.device
    idx = torch.empty(max(B, 1), dtype=torch.int64, device=dev)
    row = torch.empty(max(B, 1), dtype=torch.int64, device=dev)
    cnt = torch.empty(1, dtype=torch.int64, device=dev)  # written by the scan (or zeroed for B == 0)
    tot = torch.empty(1, dtype=torch.int64, device=dev)
    if topo is not None:
        topo = topo.to(device=dev, dtype=torch.int32).contiguous()
    wsb = int(lib.la_compact_rows_workspace(B))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    N.check(lib.la_compact_rows(first_t.data_ptr(), B, T, N.ptr(topo), table.tensor().data_ptr(), idx.data_ptr(),
                                row.data_ptr(), cnt.data_ptr(), tot.data_ptr(), ws.data_ptr(), wsb,
                                N.stream_ptr(stream)), "la_compact_rows")
    return idx, row, cnt, tot


def compact_rows_split(first_t, T: int, table: "PlanTable", topo=None, stream=None):
    """la_compact_rows_split: ascending indices of candidates with
    first_t == T, and for each its first dyad-target row and first other row
    (static joints + crank tip) in two dense row sets; device counts: items,
    target rows, other rows."""
    torch = N.require_cuda()
    lib = N.load()
    B = first_t.numel()
    dev = first_t.device
    idx, row, row2 = (torch.empty(max(B, 1), dtype=torch.int64, device=dev) for _ in range(3))
    cnt, tot, tot2 = (torch.empty(1, dtype=torch.int64, device=dev) for _ in range(3))
    if topo is not None:
        topo = topo.to(device=dev, dtype=torch.int32).contiguous()
    wsb = int(lib.la_compact_rows_split_workspace(B))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    N.check(lib.la_compact_rows_split(first_t.data_ptr(), B, T, N.ptr(topo), table.tensor().data_ptr(), idx.data_ptr(),
                                      row.data_ptr(), row2.data_ptr(), cnt.data_ptr(), tot.data_ptr(), tot2.data_ptr(),
                                      ws.data_ptr(), wsb, N.stream_ptr(stream)), "la_compact_rows_split")
    return idx, row, row2, cnt, tot, tot2


def plan_row_split(plan) -> tuple[list[int], list[int]]:
    """Joint order of the split row layout: (dyad targets ascending, other
    joints ascending) -- the static joints and the crank tip are the others."""
    targets = sorted(st.target for st in plan.steps)
    tset = set(targets)
    return targets, [j for j in range(plan.n) if j not in tset]


def plan_targets(table: "PlanTable") -> list[tuple[int, list[int]]]:
    """(n, ascending dyad targets) of every plan of a table, decoded from its
    64-byte la_plan records."""
    raw = table.host_bytes().reshape(-1, 64)
    n = raw[:, 0:2].copy().view(np.int16)[:, 0]
    ns = raw[:, 2:4].copy().view(np.int16)[:, 0]
    return [(int(n[g]), sorted(int(raw[g, 8 + 3 * s]) for s in range(int(ns[g])))) for g in range(len(raw))]


def assemble_paths(target_rows, first_row: int, pos0: np.ndarray, n: int, targets: list[int],
                   T: int = 200) -> np.ndarray:
    """Full (n, T, 2) fp32 paths of one candidate from its dyad-target rows
    (split layout: ``targets`` ascending from ``first_row``) and its f64
    pose: static joints stay at the pose (solver.py:183-184), the crank tip
    is p0 + r1 (cos, sin) with r1 = np.hypot (solver.py:180, 185-187) -- the
    f64 operations the device performs, rounded to fp32, so the rebuilt rows
    equal the device's (tests/test_gpu_solver.py)."""
    out = np.empty((n, T, 2), dtype=np.float32)
    out[targets] = np.asarray(target_rows[first_row:first_row + len(targets)])
    tset = set(targets)
    th = 2.0 * np.pi * np.arange(T) / T
    for j in range(n):
        if j in tset:
            continue
        if j == 1:
            p0 = pos0[0]
            r1 = np.hypot(pos0[1, 0] - p0[0], pos0[1, 1] - p0[1])
            out[1, :, 0] = (p0[0] + r1 * np.cos(th)).astype(np.float32)
            out[1, :, 1] = (p0[1] + r1 * np.sin(th)).astype(np.float32)
        else:
            out[j] = pos0[j].astype(np.float32)
    return out


def simulate_deferred(pos0, table: PlanTable, T: int = 200, topo=None, *, traj=None,
                      fixup_tau: float = DEFAULT_FIXUP_TAU, stream=None, timer=None,
                      dense_rows: bool = False, split_rows: bool = False, traj2=None) -> dict:
    """Two specialised launches, no host sync:

    1. fp32 screen (coarse-first, exact first lock for coarse-locked
       candidates); coarse survivors are left pending (first_t = LA_PENDING);
    2. ordered compaction of the pending candidates;
    3. f64 write-only replay of the pending ones (all T angles, exact first
       lock, fp32 paths written densely: pending item i owns rows
       [i * stride, (i + 1) * stride)); flags scattered back to the
       candidates' own slots;
    4. ordered compaction of the valid candidates.

    Returns first_t / first_joint (B,), pend_idx / pend_count (the row map of
    ``traj``), valid_idx / valid_count and traj.  ``dense_rows``: pending
    item i starts at row ``pend_row[i]`` (running sum of the plans' joint
    counts, la_compact_rows) instead of ``i * stride``, so the first
    ``pend_rows`` (device scalar) rows of ``traj`` hold every real joint path
    and no padding rows.  ``split_rows``: dense rows in two sets -- ``traj``
    holds the dyad targets' rows (pending item i from ``pend_row[i]``, its
    plan's nsteps rows in ascending joint order, ``pend_rows`` in all) and
    ``traj2`` the static joints' and crank tip's rows (``pend_row2``,
    ``pend_rows2``); see ``plan_row_split`` / ``assemble_paths``.
    """
    stages, out = _deferred_stages(pos0, table, T, topo, traj, fixup_tau, stream, dense_rows, split_rows, traj2)
    for name, fn in stages:
        fn()
        if timer:
            timer.mark(name)
    return out


def _deferred_stages(pos0, table: PlanTable, T: int, topo, traj, fixup_tau: float, stream, dense_rows: bool,
                     split_rows: bool = False, traj2=None):
    """simulate_deferred as three stage callables (screen; pending compaction
    + write pass; valid compaction) filling one result dict."""
    torch = N.require_cuda()
    B = pos0.shape[0]
    stride = table.max_n
    if traj is None:
        traj = torch.empty((max(B, 1) * stride, T, 2), dtype=torch.float32, device=pos0.device)
    if split_rows and traj2 is None:
        traj2 = torch.empty((max(B, 1) * stride, T, 2), dtype=torch.float32, device=pos0.device)
    out = {"traj": traj, "stride": stride}
    if split_rows:
        out["traj2"] = traj2

    def screen():
        out.update(simulate_tensors(pos0, table, T, topo, write_traj=False, fixup_tau=fixup_tau, stream=stream,
                                    _extra_flags=N.LA_SIM_DEFER))

    def paths():
        prow = prow2 = None
        if split_rows:
            pend, prow, prow2, pcnt, prows, prows2 = compact_rows_split(out["first_t"], N.LA_PENDING, table, topo,
                                                                        stream=stream)
            out.update(pend_row=prow, pend_rows=prows, pend_row2=prow2, pend_rows2=prows2)
        elif dense_rows:
            pend, prow, pcnt, prows = compact_rows(out["first_t"], N.LA_PENDING, table, topo, stream=stream)
            out.update(pend_row=prow, pend_rows=prows)
        else:
            pend, pcnt = compact_valid(out["first_t"], N.LA_PENDING, stream=stream)
        out.update(pend_idx=pend, pend_count=pcnt)
        simulate_tensors(pos0, table, T, topo, write_traj=True, traj=traj, traj_stride=stride, traj_row=prow,
                         cand=pend, cand_count=pcnt, fixup_tau=fixup_tau, stream=stream,
                         _extra_flags=N.LA_SIM_WRITE_ONLY | N.LA_SIM_SCATTER,
                         _outputs=(out["first_t"], out["first_joint"]), traj2=traj2, traj_row2=prow2)

    def compact():
        vidx, vcnt = compact_valid(out["first_t"], T, stream=stream)
        out.update(valid_idx=vidx, valid_count=vcnt)

    return [("screen", screen), ("paths", paths), ("compact", compact)], out


class DeferredGraph:
    """simulate_deferred captured once as CUDA graphs, one per stage, over
    fixed device buffers (pos0, topo, traj and every intermediate):
    ``replay()`` reruns the whole pipeline on the current contents of pos0 /
    topo with no host work between kernels (for repeated batches of one
    shape; results in ``out``, same keys as simulate_deferred)."""

    def __init__(self, pos0, table: PlanTable, T: int = 200, topo=None, *, traj=None,
                 fixup_tau: float = DEFAULT_FIXUP_TAU, dense_rows: bool = True, split_rows: bool = False,
                 traj2=None):
        torch = N.require_cuda()
        if topo is not None:
            topo = topo.to(device=pos0.device, dtype=torch.int32).contiguous()
        crank_table(T, pos0.device)  # device constants cached before capture
        table.tensor()
        stages, self.out = _deferred_stages(pos0, table, T, topo, traj, fixup_tau, None, dense_rows, split_rows,
                                            traj2)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up outside capture
            for _, fn in stages:
                fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graphs = []
        for name, fn in stages:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            self.graphs.append((name, g))
        self._keep = (pos0, topo)

    def replay(self, timer=None) -> dict:
        for name, g in self.graphs:
            g.replay()
            if timer:
                timer.mark(name)
        return self.out


class HostPipeline:
    """Host-to-host batch simulation: poses and plan indices in pinned host
    memory in, lock flags of every candidate and the fp32 paths of the real
    joints of every coarse survivor (dense rows) back in pinned host memory.

    The batch is split into ``chunks`` contiguous candidate ranges, each a
    DeferredGraph over its own device buffers.  Uploads run on one copy
    stream, the graphs on the compute stream, downloads on a third stream,
    so chunk c's path download (the bound: ~11 KB per valid 7-joint
    candidate over PCIe) overlaps the upload and device work of chunks
    c + 1, ...  The host waits only for each chunk's two row counts (the
    download sizes) before queueing its copies.

    ``run()`` returns host tensors (views of buffers reused by the next
    run): ``first_t`` / ``first_joint`` (B,), ``pend_idx`` (global candidate
    ids of the survivors, ascending), ``pend_row`` (each survivor's first
    row in ``traj``), ``traj`` (rows, T, 2) float32, and the byte counts of
    the step's uploads and downloads.  Rows are meaningful where
    ``first_t[pend_idx[i]] == T`` (the rest locked in the fine pass).

    ``split_rows`` (default): the device writes every joint's path, but only
    the dyad targets' rows cross PCIe -- survivor i's plan targets (ascending)
    are ``traj[pend_row[i]:]``; its static joints and crank tip are
    closed-form in the pose the host already holds (solver.py:180-187) and
    ``paths(res, i)`` rebuilds its full (n, T, 2) array bit-identical to the
    device rows.  Without it survivor i's joint j path is
    ``traj[pend_row[i] + j]``.
    """

    def __init__(self, pos_h, table: PlanTable, T: int = 200, topo_h=None, *, chunks: int = 4,
                 fixup_tau: float = DEFAULT_FIXUP_TAU, split_rows: bool = True):
        torch = N.require_cuda()
        if pos_h.is_cuda or pos_h.dtype != torch.float64 or pos_h.dim() != 3:
            raise ValueError("pos_h must be a (B, S, 2) float64 host tensor")
        if not pos_h.is_pinned():
            pos_h = pos_h.pin_memory()
        B = pos_h.shape[0]
        if topo_h is None:
            topo_h = torch.zeros(B, dtype=torch.int32)
        topo_h = topo_h.to(dtype=torch.int32).contiguous()
        if not topo_h.is_pinned():
            topo_h = topo_h.pin_memory()
        self.pos_h, self.topo_h, self.table, self.T = pos_h, topo_h, table, T
        stride = table.max_n
        chunks = max(1, min(int(chunks), B))
        bounds = [B * c // chunks for c in range(chunks + 1)]
        self.ranges = [(bounds[c], bounds[c + 1]) for c in range(chunks) if bounds[c + 1] > bounds[c]]
        self.pos_d = torch.empty(pos_h.shape, dtype=pos_h.dtype, device="cuda")
        self.topo_d = torch.empty(topo_h.shape, dtype=topo_h.dtype, device="cuda")
        self.pos_d.copy_(pos_h)
        self.topo_d.copy_(topo_h)
        self.graphs = []
        self.split = bool(split_rows)
        for lo, hi in self.ranges:
            traj = torch.empty(((hi - lo) * stride, T, 2), dtype=torch.float32, device="cuda")
            traj2 = torch.empty(((hi - lo) * stride, T, 2), dtype=torch.float32, device="cuda") if self.split else None
            self.graphs.append(DeferredGraph(self.pos_d[lo:hi], table, T, self.topo_d[lo:hi], traj=traj,
                                             fixup_tau=fixup_tau, split_rows=self.split, traj2=traj2))
        self._targets = plan_targets(table) if self.split else None
        nc = len(self.ranges)
        self.cnt_d = torch.empty((nc, 2), dtype=torch.int64, device="cuda")
        self.cnt_h = torch.empty((nc, 2), dtype=torch.int64).pin_memory()
        self.ft_h = torch.empty(B, dtype=torch.int32).pin_memory()
        self.fj_h = torch.empty(B, dtype=torch.int32).pin_memory()
        self.idx_h = torch.empty(B, dtype=torch.int64).pin_memory()
        self.row_h = torch.empty(B, dtype=torch.int64).pin_memory()
        self.traj_h = torch.empty((B * stride, T, 2), dtype=torch.float32).pin_memory()
        self.up = torch.cuda.Stream()
        self.down = torch.cuda.Stream()
        self.ev_in = [torch.cuda.Event() for _ in self.ranges]
        self.ev_done = [torch.cuda.Event() for _ in self.ranges]
        self.ev_cnt = [torch.cuda.Event() for _ in self.ranges]

    def run(self) -> dict:
        torch = N.require_cuda()
        comp = torch.cuda.current_stream()
        self.up.wait_stream(comp)  # previous users of the input buffers
        self.down.wait_stream(comp)
        with torch.cuda.stream(self.up):
            for (lo, hi), ev in zip(self.ranges, self.ev_in):
                self.pos_d[lo:hi].copy_(self.pos_h[lo:hi], non_blocking=True)
                self.topo_d[lo:hi].copy_(self.topo_h[lo:hi], non_blocking=True)
                ev.record(self.up)
        outs = []
        for c, g in enumerate(self.graphs):
            comp.wait_event(self.ev_in[c])
            out = g.replay()
            self.cnt_d[c, 0:1].copy_(out["pend_count"])
            self.cnt_d[c, 1:2].copy_(out["pend_rows"])
            self.cnt_h[c].copy_(self.cnt_d[c], non_blocking=True)
            self.ev_cnt[c].record(comp)
            outs.append(out)
        nrow = npend = 0
        down_rows = []
        for c, ((lo, hi), out) in enumerate(zip(self.ranges, outs)):
            self.ev_cnt[c].synchronize()
            p, r = int(self.cnt_h[c, 0]), int(self.cnt_h[c, 1])
            self.down.wait_event(self.ev_cnt[c])
            with torch.cuda.stream(self.down):
                self.traj_h[nrow:nrow + r].copy_(out["traj"][:r], non_blocking=True)
                self.ft_h[lo:hi].copy_(out["first_t"], non_blocking=True)
                self.fj_h[lo:hi].copy_(out["first_joint"], non_blocking=True)
                self.idx_h[npend:npend + p].copy_(out["pend_idx"][:p], non_blocking=True)
                self.row_h[npend:npend + p].copy_(out["pend_row"][:p], non_blocking=True)
            down_rows.append((lo, nrow, npend, p))
            nrow += r
            npend += p
        self.down.synchronize()
        for lo, r0, p0, p in down_rows:  # chunk-local ids and rows -> global
            if lo:
                self.idx_h[p0:p0 + p] += lo
            if r0:
                self.row_h[p0:p0 + p] += r0
        comp.wait_stream(self.down)
        B = self.pos_h.shape[0]
        return {"first_t": self.ft_h, "first_joint": self.fj_h, "pend_idx": self.idx_h[:npend],
                "pend_row": self.row_h[:npend], "traj": self.traj_h[:nrow], "split_rows": self.split,
                "h2d_bytes": self.pos_h.numel() * 8 + self.topo_h.numel() * 4,
                "d2h_bytes": B * 8 + len(self.ranges) * 16 + nrow * self.T * 8 + npend * 16}

    def paths(self, res: dict, i: int) -> np.ndarray:
        """Full (n, T, 2) fp32 paths of survivor i of a ``run()`` result."""
        b = int(res["pend_idx"][i])
        g = int(self.topo_h[b])
        row = int(res["pend_row"][i])
        if not self.split:
            n = self._n_of(g)
            return res["traj"][row:row + n].numpy()
        n, targets = self._targets[g]
        return assemble_paths(res["traj"], row, self.pos_h[b].numpy(), n, targets, self.T)

    def _n_of(self, g: int) -> int:
        return int(self.table.host_bytes().reshape(-1, 64)[g, 0:2].copy().view(np.int16)[0])


def simulate_compact(pos0, table: PlanTable, T: int = 200, topo=None, *, traj=None, traj_f64: bool = False,
                     fixup_tau: float = DEFAULT_FIXUP_TAU, stream=None) -> dict:
    """Batch simulation with compacted output, all on device, no host sync.

    1. screen every candidate (fp32 + f64 fix-up, coarse-first, exact
       first lock) -> first_t / first_joint;
    2. ordered compaction of the valid ones (la_compact_valid);
    3. replay only the valid candidates in f64 over all T angles, writing
       their paths densely: valid candidate v occupies rows
       [v * stride, (v + 1) * stride) of ``traj``.

    Returns first_t, first_joint (B,), valid_idx (B,) int64 (first
    ``valid_count`` entries meaningful), valid_count (1,) int64 (device) and
    traj ((B * stride, T, 2) worst-case buffer).
    """
    torch = N.require_cuda()
    B, S, _ = pos0.shape
    stride = table.max_n
    res = simulate_tensors(pos0, table, T, topo, write_traj=False, fixup_tau=fixup_tau, stream=stream,
                           exact=traj_f64)
    idx, cnt = compact_valid(res["first_t"], T, stream=stream)
    if traj is None:
        traj = torch.empty((max(B, 1) * stride, T, 2), dtype=torch.float64 if traj_f64 else torch.float32,
                           device=pos0.device)
    simulate_tensors(pos0, table, T, topo, write_traj=True, traj=traj, traj_stride=stride, traj_f64=traj_f64,
                     cand=idx, cand_count=cnt, coarse=False, fixup_tau=fixup_tau, stream=stream)
    res.update(valid_idx=idx, valid_count=cnt, traj=traj, stride=stride)
    return res


# ------------------------------------------------------------ drop-in API
def plan_geometry(plan: SolutionPlan, positions0: np.ndarray):
    """Per-step r_a, r_b, branch for one pose (solver.py:105-120), on device."""
    torch = N.require_cuda()
    lib = N.load()
    pos = np.ascontiguousarray(np.asarray(positions0, dtype=np.float64))
    S = len(plan.steps)
    if S == 0:
        e = np.zeros(0)
        return e, e.copy(), e.copy()
    table = PlanTable([plan])
    dpos = torch.from_numpy(np.array(pos, dtype=np.float64).reshape(1, -1, 2)).cuda()
    outs = [torch.empty((1, N.LA_MAX_STEPS), dtype=torch.float64, device=dpos.device) for _ in range(3)]
    N.check(lib.la_plan_geometry(dpos.data_ptr(), None, table.tensor().data_ptr(), 1, 1, pos.shape[0],
                                 outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(),
                                 N.stream_ptr()), "la_plan_geometry")
    r_a, r_b, br = (o[0, :S].cpu().numpy() for o in outs)
    return r_a, r_b, br


def dyad_solve(p_a, p_b, r_a: float, r_b: float, branch: float):
    """Circle-circle intersection (solver.py:123-139) via la_dyad_solve.

    Returns an (x, y) tuple or None when the circles do not meet.
    """
    torch = N.require_cuda()
    lib = N.load()
    dev = torch.device("cuda")
    pa = torch.tensor([[float(p_a[0]), float(p_a[1])]], dtype=torch.float64, device=dev)
    pb = torch.tensor([[float(p_b[0]), float(p_b[1])]], dtype=torch.float64, device=dev)
    ra = torch.tensor([float(r_a)], dtype=torch.float64, device=dev)
    rb = torch.tensor([float(r_b)], dtype=torch.float64, device=dev)
    br = torch.tensor([float(branch)], dtype=torch.float64, device=dev)
    out = torch.empty((1, 2), dtype=torch.float64, device=dev)
    ok = torch.empty(1, dtype=torch.int32, device=dev)
    N.check(lib.la_dyad_solve(pa.data_ptr(), pb.data_ptr(), ra.data_ptr(), rb.data_ptr(), br.data_ptr(), 1,
                              out.data_ptr(), ok.data_ptr(), N.stream_ptr()), "la_dyad_solve")
    if int(ok.item()) == 0:
        return None
    o = out.cpu().numpy()[0]
    return (float(o[0]), float(o[1]))


def _outcomes(res: dict, T: int, n: int) -> list[SimOutcome]:
    ft = res["first_t"].cpu().numpy()
    fj = res["first_joint"].cpu().numpy()
    traj = res.get("traj")
    P = None
    if traj is not None and (ft == T).any():
        P = traj.view(-1, n, T, 2).cpu().numpy().astype(np.float64, copy=False)
    outs: list[SimOutcome] = []
    for b in range(len(ft)):
        if ft[b] < T:
            outs.append(Locking(step=int(ft[b]), joint=int(fj[b])))
        else:
            outs.append(Trajectory(P[b]))
    return outs


def simulate_batch(positions0_batch: np.ndarray, plan: SolutionPlan, T: int = 200, *,
                   fixup_tau: float = DEFAULT_FIXUP_TAU) -> list[SimOutcome]:
    """Replay one plan over a batch of poses (solver.py:172-239) on the GPU.

    Trajectories are computed in f64 on the device in the reference's
    operation order and returned as (n, T, 2) float64 arrays; lock flags
    follow the reference rule (fp32 screen with f64 replay near any lock).
    """
    torch = N.require_cuda()
    pos = np.asarray(positions0_batch, dtype=np.float64)
    if pos.ndim != 3 or pos.shape[2] != 2:
        raise ValueError("positions0_batch must be (B, n, 2)")
    B, n, _ = pos.shape
    if B == 0:
        return []
    dpos = torch.from_numpy(np.array(pos, dtype=np.float64, order="C")).cuda()
    res = simulate_tensors(dpos, PlanTable([plan]), T, write_traj=True, traj_stride=n, fixup_tau=fixup_tau,
                           traj_f64=True)
    return _outcomes(res, T, n)


def simulate(mech: Mechanism, plan: SolutionPlan, T: int = 200) -> SimOutcome:
    """Single-mechanism replay (solver.py:142-169): a batch of one."""
    return simulate_batch(mech.positions0[None, :, :], plan, T)[0]


def check_feasible(mech: Mechanism, plan: SolutionPlan, T_low: int = 50, T_high: int = 200) -> bool:
    """Two-fidelity gate (solver.py:242-249): T_low sweep, then T_high."""
    torch = N.require_cuda()
    dpos = torch.from_numpy(np.ascontiguousarray(mech.positions0[None, :, :], dtype=np.float64)).cuda()
    table = PlanTable([plan])
    if T_high == 4 * T_low:
        # the T_low angles are every 4th T_high angle (bit-identical thetas):
        # one coarse-first launch answers both sweeps
        res = simulate_tensors(dpos, table, T_high, write_traj=False, low=True, exact=True)
        return bool(int(res["low_t"].item()) < 0 and int(res["first_t"].item()) == T_high)
    lo = simulate_tensors(dpos, table, T_low, write_traj=False, exact=True)
    if int(lo["first_t"].item()) < T_low:
        return False
    hi = simulate_tensors(dpos, table, T_high, write_traj=False, exact=True)
    return int(hi["first_t"].item()) == T_high
