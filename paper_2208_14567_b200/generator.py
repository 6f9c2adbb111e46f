"""Rejection-sampling driver around the GPU validity screen.

Reference: linkatlas generator.py.  Topology growth (generator.py:156-222)
runs in the native generator (csrc/gen.cpp) on the caller's PCG64 state and
candidate-pose sampling (generator.py:225-238) draws from numpy, both
consuming the streams exactly as the reference does, so seeded runs produce
the same topologies and poses.  The two-fidelity gate inside ``find_valid_variant``
(generator.py:241-283: T_low = 50 sweep, survivors confirmed at T_high =
200) runs on the device: one coarse-first ``la_simulate`` launch screens a
whole look-ahead window of candidate batches, and the host walks the flags
in stream order to reproduce ``attempts`` and the negative-sample draws bit
for bit.  The pose stream is drawn ahead and rewound so the caller's RNG
ends in the same state as after the reference loop.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from paper_2208_14567_b200 import _native as N
from paper_2208_14567_b200.mechanism import ARM_PIVOT, ARM_TIP, Mechanism
from paper_2208_14567_b200.solver import PlanTable, SolutionPlan, Trajectory, compile_order, simulate_tensors

NMAX = N.LA_MAX_JOINTS


class GenerationError(RuntimeError):
    pass


@dataclass
class GenerationConfig:
    """generator.py:31-57."""

    count: int
    n_min: int = 8
    n_max: int = 20
    ng_probability: float = 0.25
    variants_per_topology: int = 5
    T_low: int = 50
    T_high: int = 200
    max_attempts: int = 5000
    seed: int = 0
    workers: int = 1
    negative_rate: float = 0.0
    topology_retries: int = 1000
    batch: int = 256

    def __post_init__(self):
        if self.n_min < 4:
            raise ValueError("n_min must be >= 4")
        if self.n_max < self.n_min:
            raise ValueError("n_max < n_min")
        if self.variants_per_topology < 1:
            raise ValueError("variants_per_topology must be >= 1")
        if not self.T_low < self.T_high:
            raise ValueError("T_low must be < T_high")
        if self.max_attempts < 1:
            raise ValueError("max_attempts must be >= 1")


@dataclass
class GenerationStats:
    """Mergeable tallies keyed by joint count (generator.py:60-131)."""

    simulated_by_n: dict[int, int] = field(default_factory=dict)
    accepted_by_n: dict[int, int] = field(default_factory=dict)
    attempts_samples: dict[int, list[int]] = field(default_factory=dict)
    topologies_discarded: int = 0

    @property
    def simulated(self) -> int:
        return sum(self.simulated_by_n.values())

    @property
    def accepted(self) -> int:
        return sum(self.accepted_by_n.values())

    @property
    def locking(self) -> int:
        return self.simulated - self.accepted

    def record_success(self, n: int, attempts: int) -> None:
        self.simulated_by_n[n] = self.simulated_by_n.get(n, 0) + attempts
        self.accepted_by_n[n] = self.accepted_by_n.get(n, 0) + 1
        self.attempts_samples.setdefault(n, []).append(attempts)

    def record_failure(self, n: int, attempts: int) -> None:
        self.simulated_by_n[n] = self.simulated_by_n.get(n, 0) + attempts

    def mean_attempts(self, n: int) -> float:
        acc = self.accepted_by_n.get(n, 0)
        return math.nan if acc == 0 else self.simulated_by_n.get(n, 0) / acc

    def median_attempts(self, n: int) -> float:
        s = self.attempts_samples.get(n, [])
        return float(np.median(s)) if s else math.nan

    def rejection_rate(self, n: int) -> float:
        sim = self.simulated_by_n.get(n, 0)
        return math.nan if sim == 0 else 1.0 - self.accepted_by_n.get(n, 0) / sim

    def merge(self, other: "GenerationStats") -> None:
        for n, v in other.simulated_by_n.items():
            self.simulated_by_n[n] = self.simulated_by_n.get(n, 0) + v
        for n, v in other.accepted_by_n.items():
            self.accepted_by_n[n] = self.accepted_by_n.get(n, 0) + v
        for n, v in other.attempts_samples.items():
            self.attempts_samples.setdefault(n, []).extend(v)
        self.topologies_discarded += other.topologies_discarded


@dataclass
class NegativeSample:
    mechanism: Mechanism
    locking_step: int


@dataclass
class VariantResult:
    mechanism: Mechanism
    trajectory: Trajectory
    attempts: int


# ------------------------------------------------------------ topology (native)
_M64 = (1 << 64) - 1


def sample_topology(rng: np.random.Generator, n: int, ng_probability: float = 0.25,
                    retries: int = 1000) -> tuple[Mechanism, SolutionPlan]:
    """generator.py:200-222 on the caller's Generator: the native topology
    operator (csrc/gen.cpp, la_sample_topology_rng: constrained growth with
    terminal tracking, plan compile, last-joint checks) runs on a copy of
    ``rng``'s PCG64 state, which is then written back, so the stream
    advances exactly as the reference's draws advance it."""
    bg = rng.bit_generator
    stt = bg.state
    if stt.get("bit_generator") != "PCG64":
        raise TypeError("sample_topology needs a PCG64-backed Generator (numpy's default_rng)")
    lib = N.load()
    s, inc = int(stt["state"]["state"]), int(stt["state"]["inc"])
    st = np.array([s >> 64, s & _M64, inc >> 64, inc & _M64], dtype=np.uint64)
    buf = np.array([int(stt["has_uint32"]), int(stt["uinteger"])], dtype=np.uint32)
    rec = N.LaPlan()
    types = np.zeros(NMAX, dtype=np.int8)
    adj = np.zeros((NMAX, NMAX), dtype=np.uint8)
    rc = lib.la_sample_topology_rng(st.ctypes.data, buf.ctypes.data, int(n), float(ng_probability), int(retries),
                                    C.addressof(rec), types.ctypes.data, adj.ctypes.data)
    stt["state"]["state"] = (int(st[0]) << 64) | int(st[1])
    stt["has_uint32"], stt["uinteger"] = int(buf[0]), int(buf[1])
    bg.state = stt
    if rc == N.LA_ERANGE:
        raise GenerationError(f"no valid topology with n={n} after {retries} tries")
    N.check(rc, "la_sample_topology_rng")
    pos = np.full((n, 2), np.nan)
    pos[0], pos[1] = ARM_PIVOT, ARM_TIP
    mech = Mechanism(adj[:n, :n].copy(), types[:n].copy(), pos)
    fixed, steps = compile_order(mech.adjacency, mech.types)
    return mech, SolutionPlan(mech.n, fixed, steps, None, None, None)


def sample_positions(topology: Mechanism, rng: np.random.Generator) -> np.ndarray:
    """generator.py:225-231."""
    pos = rng.uniform(size=(topology.n, 2))
    pos[0] = ARM_PIVOT
    pos[1] = ARM_TIP
    return pos


def _sample_positions_batch(n: int, k: int, rng: np.random.Generator) -> np.ndarray:
    """generator.py:234-238."""
    pos = rng.uniform(size=(k, n, 2))
    pos[:, 0] = ARM_PIVOT
    pos[:, 1] = ARM_TIP
    return pos


# ------------------------------------------------------------ native streams
def native_topologies(seed: int, G: int, n_lo: int, n_hi: int, *, g0: int = 0, ng_probability: float = 0.25,
                      retries: int = 1000, threads: int = 0):
    """G generator topologies, group g drawn exactly like
    ``n = default_rng([seed, g0+g, 0]).integers(n_lo, n_hi+1)`` followed by
    ``sample_topology`` on the same stream — by the native multi-threaded
    generator (csrc/gen.cpp).  Returns (la_plan bytes (G*64,) uint8, types
    (G, 20) int8, adjacency (G, 20, 20) uint8, n (G,) int32)."""
    import os as _os

    lib = N.load()
    plans = np.zeros(G * 64, dtype=np.uint8)
    types = np.zeros((G, N.LA_MAX_JOINTS), dtype=np.int8)
    adj = np.zeros((G, N.LA_MAX_JOINTS, N.LA_MAX_JOINTS), dtype=np.uint8)
    ns = np.zeros(G, dtype=np.int32)
    th = threads or len(_os.sched_getaffinity(0))
    N.check(lib.la_sample_topologies(int(seed), int(g0), int(G), int(n_lo), int(n_hi), float(ng_probability),
                                     int(retries), int(th), plans.ctypes.data, types.ctypes.data, adj.ctypes.data,
                                     ns.ctypes.data), "la_sample_topologies")
    return plans, types, adj, ns


def native_poses(seed: int, n_of_group: np.ndarray, per_group: int, stride: int, *, g0: int = 0,
                 threads: int = 0) -> np.ndarray:
    """(G*per_group, stride, 2) float64 poses: group g is
    ``_sample_positions_batch(n_g, per_group, default_rng([seed, g0+g, 1]))``
    padded with NaN, drawn by the native generator."""
    import os as _os

    lib = N.load()
    ng = np.ascontiguousarray(n_of_group, dtype=np.int32)
    out = np.empty((len(ng) * per_group, stride, 2), dtype=np.float64)
    th = threads or len(_os.sched_getaffinity(0))
    N.check(lib.la_sample_poses(int(seed), int(g0), len(ng), int(per_group), ng.ctypes.data, int(stride), int(th),
                                out.ctypes.data), "la_sample_poses")
    return out


# ------------------------------------------------------------ GPU gate driver
def find_valid_variant(topology: Mechanism, plan: SolutionPlan, rng: np.random.Generator,
                       max_attempts: int = 5000, T_low: int = 50, T_high: int = 200, batch: int = 256,
                       negative_rate: float = 0.0, neg_rng: np.random.Generator | None = None,
                       negatives: list[NegativeSample] | None = None, lookahead: int = 16) -> VariantResult | None:
    """Rejection-sample poses until one passes the two-fidelity gate
    (generator.py:241-283); returns the accepted mechanism, its T_high
    trajectory and the number of candidates consumed, or None at the cap."""
    torch = N.require_cuda()
    n = topology.n
    table = PlanTable([plan])
    fused = T_high == 4 * T_low
    consumed = 0
    while consumed < max_attempts:
        # draw a look-ahead window of whole reference batches in one go
        sizes = []
        left = max_attempts - consumed
        for _ in range(max(1, lookahead)):
            if left <= 0:
                break
            sizes.append(min(batch, left))
            left -= sizes[-1]
        state = rng.bit_generator.state
        chunks = [_sample_positions_batch(n, k, rng) for k in sizes]
        cand = np.concatenate(chunks)
        dpos = torch.from_numpy(cand).cuda()
        if fused:
            res = simulate_tensors(dpos, table, T_high, write_traj=False, low=True, exact=True)
            low_t = res["low_t"].cpu().numpy()
            high_ok = res["first_t"].cpu().numpy() == T_high
        else:
            lo = simulate_tensors(dpos, table, T_low, write_traj=False, exact=True)
            hi = simulate_tensors(dpos, table, T_high, write_traj=False, exact=True)
            ft = lo["first_t"].cpu().numpy()
            low_t = np.where(ft < T_low, ft, -1)
            high_ok = hi["first_t"].cpu().numpy() == T_high
        base = 0
        for bi, k in enumerate(sizes):
            for idx in range(k):
                g = base + idx
                if low_t[g] >= 0:
                    if negatives is not None and negative_rate > 0.0 and neg_rng is not None:
                        if neg_rng.random() < negative_rate:
                            negatives.append(NegativeSample(topology.with_positions(cand[g]), int(low_t[g])))
                    continue
                if not high_ok[g]:
                    continue
                # success: rewind the pose stream to the end of this batch
                rng.bit_generator.state = state
                for kk in sizes[:bi + 1]:
                    _sample_positions_batch(n, kk, rng)
                traj = _trajectory(cand[g], table, T_high)
                return VariantResult(mechanism=topology.with_positions(cand[g]), trajectory=traj,
                                     attempts=consumed + idx + 1)
            consumed += k
            base += k
    return None


def _trajectory(pos: np.ndarray, table: PlanTable, T: int) -> Trajectory:
    torch = N.require_cuda()
    dpos = torch.from_numpy(np.ascontiguousarray(pos[None])).cuda()
    res = simulate_tensors(dpos, table, T, write_traj=True, traj_stride=pos.shape[0], traj_f64=True)
    return Trajectory(res["traj"].view(pos.shape[0], T, 2).cpu().numpy())


# ------------------------------------------------------------ dataset generation
@dataclass
class GeneratedRecord:
    """generator.py:148-153."""

    slot: int
    variant: int
    mechanism: Mechanism
    trajectory: Trajectory
    attempts: int


@dataclass
class GeneratedBlock:
    """Records of a block of slots as arrays (slot order): meta (R, 4) =
    slot, variant, attempts, n; pos0 (R, 20, 2); adjacency (R, 20, 20);
    types (R, 20); traj (sum n, T_high, 2) f64 with record i in rows
    row0[i]:row0[i+1] (a CUDA tensor with ``traj_on_device``, for pipelines
    that normalise and index the paths without a host round trip)."""

    meta: np.ndarray
    pos0: np.ndarray
    adjacency: np.ndarray
    types: np.ndarray
    traj: np.ndarray
    row0: np.ndarray

    @property
    def R(self) -> int:
        return len(self.meta)

    def record(self, i: int) -> GeneratedRecord:
        slot, variant, attempts, n = (int(x) for x in self.meta[i])
        mech = Mechanism(self.adjacency[i, :n, :n].copy(), self.types[i, :n].copy(), self.pos0[i, :n].copy())
        t = self.traj[self.row0[i]:self.row0[i + 1]]
        if not isinstance(t, np.ndarray):
            t = t.cpu().numpy()
        return GeneratedRecord(slot, variant, mech, Trajectory(t), attempts)


def _mechanisms(adj: np.ndarray, types: np.ndarray, pos: np.ndarray, n: np.ndarray) -> list[Mechanism]:
    return [Mechanism(adj[i, :n[i], :n[i]].copy(), types[i, :n[i]].astype(np.int8), pos[i, :n[i]].copy())
            for i in range(len(n))]


_PINNED: dict = {}


def _pinned(torch, key, shape, dtype):
    """Reusable pinned host buffer (cudaHostAlloc is slow; generation runs
    allocate the same window buffers block after block)."""
    t = _PINNED.get(key)
    if t is None or t.dtype != dtype or t.numel() < int(np.prod(shape)):
        t = torch.empty(int(np.prod(shape)), dtype=dtype).pin_memory()
        _PINNED[key] = t
    return t[:int(np.prod(shape))].view(*shape)


class _EngineLane:
    """One la_gen engine with its own buffers and CUDA stream (GenerationRun
    internals): submit() lays out the next window on the host and queues
    poses -> gate -> flags D2H on the stream; wait_and_consume() waits for
    that window and walks its flags."""

    def __init__(self, run, lib, torch, dev, slot0: int, nslots: int, index: int = 0):
        import os as _os

        self.run, self.lib, self.torch, self.dev = run, lib, torch, dev
        c = run.config
        self.c = c
        cfg = run._cfg()
        self.eng = lib.la_gen_create(C.byref(cfg), int(slot0), int(nslots))
        if not self.eng:
            raise ValueError(N.last_error())
        self.th = run.threads or len(_os.sched_getaffinity(0))
        self.fused = c.T_high == 4 * c.T_low
        self.stream = torch.cuda.Stream(device=dev)
        self.per_window = min(run.window_cap, max(c.batch, nslots * run.lookahead * c.batch))
        self.stride = int(c.n_max)
        self.plans_h = np.zeros((max(nslots, 1), 64), dtype=np.uint8)
        self.flags_h = _pinned(torch, ("flags", index), (2, self.per_window), torch.int32)
        self.n_plans = C.c_int32(0)
        self.pos_d = torch.empty((self.per_window, self.stride, 2), dtype=torch.float64, device=dev)
        self.topo_d = torch.empty(self.per_window, dtype=torch.int32, device=dev)
        self.max_b = max(nslots * run.lookahead, 1)
        if run.device_poses:
            self.desc_h = _pinned(torch, ("desc", index), (self.max_b, C.sizeof(N.LaGenBatch)), torch.uint8)
            self.desc_d = torch.empty_like(self.desc_h, device=dev)
            self.nb = C.c_int64(0)
        else:
            self.pos_h = _pinned(torch, ("pos", index), (self.per_window, NMAX, 2), torch.float64)
            self.plan_h = _pinned(torch, ("plan", index), (self.per_window,), torch.int32)
        # fused gate: one la_simulate per window straight from preallocated
        # buffers (plan records through a pinned staging buffer)
        self.plans_p = _pinned(torch, ("plans", index), (max(nslots, 1) * 64,), torch.uint8)
        self.plans_d = torch.empty(max(nslots, 1) * 64, dtype=torch.uint8, device=dev)
        self.flags_d = torch.empty((4, self.per_window), dtype=torch.int32, device=dev)
        from paper_2208_14567_b200.solver import DEFAULT_FIXUP_TAU, crank_table

        self.cs = crank_table(c.T_high, dev)
        self.args = N.LaSimArgs()
        a = self.args
        a.pos0, a.topo, a.plans, a.crank_cs = self.pos_d.data_ptr(), self.topo_d.data_ptr(), \
            self.plans_d.data_ptr(), self.cs.data_ptr()
        a.pos_stride, a.T, a.traj_stride = self.stride, c.T_high, self.stride
        a.first_t, a.first_joint = self.flags_d[0].data_ptr(), self.flags_d[1].data_ptr()
        a.low_t, a.low_joint = self.flags_d[2].data_ptr(), self.flags_d[3].data_ptr()
        a.fixup_tau = float(DEFAULT_FIXUP_TAU)
        a.flags = N.LA_SIM_GATE_ONLY | N.LA_SIM_EXACT64
        self.active = True
        self.m = 0
        self.done = None
        self.keep = None

    def submit(self):
        run, lib, torch, c = self.run, self.lib, self.torch, self.c
        t0 = time.perf_counter()
        if run.device_poses:
            m = lib.la_gen_window_dev(self.eng, run.lookahead, self.per_window, self.desc_h.data_ptr(), self.max_b,
                                      C.byref(self.nb), self.plans_h.ctypes.data, C.byref(self.n_plans))
        else:
            m = lib.la_gen_window(self.eng, run.lookahead, self.per_window, self.th, self.pos_h.data_ptr(),
                                  self.plan_h.data_ptr(), self.plans_h.ctypes.data, C.byref(self.n_plans))
        if m < 0:
            raise GenerationError(N.last_error())
        run.timings["window"] += time.perf_counter() - t0
        if m == 0:
            self.active = False
            return
        self.m = int(m)
        t1 = time.perf_counter()
        np_ = self.n_plans.value
        if self.fused and run.device_poses:
            with torch.cuda.stream(self.stream):
                sp = N.stream_ptr(self.stream)
                nb = self.nb.value
                self.plans_p[:np_ * 64].numpy()[:] = self.plans_h[:np_].reshape(-1)
                self.plans_d[:np_ * 64].copy_(self.plans_p[:np_ * 64], non_blocking=True)
                self.desc_d[:nb].copy_(self.desc_h[:nb], non_blocking=True)
                N.check(self.lib.la_gen_poses(self.desc_d.data_ptr(), nb, self.stride, self.pos_d.data_ptr(),
                                              self.topo_d.data_ptr(), sp), "la_gen_poses")
                self.args.B, self.args.G = int(m), int(np_)
                N.check(self.lib.la_simulate(self.args, sp), "la_simulate")
                self.flags_h[0, :m].copy_(self.flags_d[0, :m], non_blocking=True)
                self.flags_h[1, :m].copy_(self.flags_d[2, :m], non_blocking=True)
                self.done = torch.cuda.Event()
                self.done.record(self.stream)
            run.timings["enqueue"] = run.timings.get("enqueue", 0.0) + time.perf_counter() - t1
            return
        ns = self.plans_h[:np_, :2].copy().view(np.int16)[:, 0].astype(np.int32)
        with torch.cuda.stream(self.stream):
            table = PlanTable.from_records(self.plans_h[:np_].reshape(-1).copy(), ns, device=self.dev)
            pd, topo = self.pos_d[:m], self.topo_d[:m]
            sp = N.stream_ptr(self.stream)
            if run.device_poses:
                nb = self.nb.value
                self.desc_d[:nb].copy_(self.desc_h[:nb], non_blocking=True)
                N.check(self.lib.la_gen_poses(self.desc_d.data_ptr(), nb, self.stride, pd.data_ptr(), topo.data_ptr(),
                                              sp), "la_gen_poses")
            else:
                pd.copy_(self.pos_h[:m, :self.stride], non_blocking=True)
                topo.copy_(self.plan_h[:m], non_blocking=True)
            if self.fused:
                res = simulate_tensors(pd, table, c.T_high, topo, write_traj=False, low=True, gate_only=True,
                                       exact=True, stream=self.stream)
                self.flags_h[0, :m].copy_(res["first_t"], non_blocking=True)
                self.flags_h[1, :m].copy_(res["low_t"], non_blocking=True)
            else:
                lo = simulate_tensors(pd, table, c.T_low, topo, write_traj=False, exact=True, stream=self.stream)
                hi = simulate_tensors(pd, table, c.T_high, topo, write_traj=False, exact=True, stream=self.stream)
                self.flags_h[0, :m].copy_(hi["first_t"], non_blocking=True)
                ft = lo["first_t"]
                self.flags_h[1, :m].copy_(torch.where(ft < c.T_low, ft, torch.full_like(ft, -1)), non_blocking=True)
            self.keep = (table, res if self.fused else (lo, hi))  # alive until the stream is done
            self.done = torch.cuda.Event()
            self.done.record(self.stream)
        run.timings["enqueue"] = run.timings.get("enqueue", 0.0) + time.perf_counter() - t1

    def wait_and_consume(self):
        run = self.run
        t0 = time.perf_counter()
        self.done.synchronize()
        t1 = time.perf_counter()
        run.timings["device"] += t1 - t0
        run.windows += 1
        run.screened += self.m
        src = None if run.device_poses else self.pos_h.data_ptr()
        rc = self.lib.la_gen_consume(self.eng, src, self.flags_h[0].data_ptr(), self.flags_h[1].data_ptr())
        if rc != 0:
            raise GenerationError(N.last_error())
        self.keep = None
        run.timings["consume"] += time.perf_counter() - t1

    def results(self):
        lib, eng = self.lib, self.eng
        R = lib.la_gen_count(eng, 0)
        meta = np.zeros((R, 4), dtype=np.int64)
        rpos = np.zeros((R, NMAX, 2))
        rplans = np.zeros((R, 64), dtype=np.uint8)
        radj = np.zeros((R, NMAX, NMAX), dtype=np.uint8)
        rtypes = np.zeros((R, NMAX), dtype=np.int8)
        N.check(lib.la_gen_records(eng, meta.ctypes.data, rpos.ctypes.data, rplans.ctypes.data, radj.ctypes.data,
                                   rtypes.ctypes.data), "la_gen_records")
        Q = lib.la_gen_count(eng, 1)
        nmeta = np.zeros((Q, 3), dtype=np.int64)
        npos = np.zeros((Q, NMAX, 2))
        nadj = np.zeros((Q, NMAX, NMAX), dtype=np.uint8)
        ntypes = np.zeros((Q, NMAX), dtype=np.int8)
        N.check(lib.la_gen_negatives(eng, nmeta.ctypes.data, npos.ctypes.data, nadj.ctypes.data,
                                     ntypes.ctypes.data), "la_gen_negatives")
        by_n = np.zeros((NMAX + 1, 2), dtype=np.int64)
        disc = C.c_int64(0)
        N.check(lib.la_gen_stats(eng, by_n.ctypes.data, C.byref(disc)), "la_gen_stats")
        return meta, rpos, rplans, radj, rtypes, nmeta, npos, nadj, ntypes, by_n, int(disc.value)

    def close(self):
        if self.eng:
            if self.done is not None:
                self.done.synchronize()
            self.lib.la_gen_destroy(self.eng)
            self.eng = None


class GenerationRun:
    """Dataset generation (generator.py:336-375) with the slot loop in the
    native engine and the two-fidelity gate on the GPU.

    Each block of slots is one ``la_gen_*`` engine: it draws look-ahead
    windows of whole reference batches from copies of every searching slot's
    pose stream, one ``la_simulate`` launch (gate mode, coarse T_low lock
    step) screens the window, and the engine walks the flags in each slot's
    stream order.  Records, ``attempts``, negatives and stats are identical to
    the reference run with ``workers=1`` (records come out in slot order for
    any ``workers``; the reference's pool order is not deterministic).
    Trajectories of accepted variants are f64 T_high paths from la_simulate.
    """

    def __init__(self, config: GenerationConfig, *, lookahead: int = 4, slot_block: int = 1 << 14,
                 window_cap: int = 1 << 21, threads: int | None = None, device=None, device_poses: bool = True,
                 traj_on_device: bool = False, slot_range: tuple[int, int] | None = None,
                 overlap: bool = True):
        self.config = config
        self.stats = GenerationStats()
        self.negatives: list[NegativeSample] = []
        self.lookahead = int(lookahead)
        self.slot_block = int(slot_block)
        self.window_cap = int(window_cap)
        self.threads = threads
        self.device = device
        self.overlap = bool(overlap)  # two engines ping-ponged on two streams
        self.slot_range = slot_range  # (first, end) slots of this shard; records() then cuts at count per shard
        self.traj_on_device = bool(traj_on_device)  # GeneratedBlock.traj stays a CUDA tensor
        self.device_poses = bool(device_poses)  # poses drawn by la_gen_poses (else host threads + H2D)
        self.timings = {"window": 0.0, "device": 0.0, "consume": 0.0, "finish": 0.0}  # host wall seconds
        self.windows = 0         # GPU launches of the gate
        self.screened = 0        # candidates screened on the GPU (>= stats.simulated)

    def _cfg(self) -> N.LaGenCfg:
        c = self.config
        return N.LaGenCfg(int(c.seed), int(c.n_min), int(c.n_max), float(c.ng_probability),
                          int(c.variants_per_topology), int(c.T_low), int(c.T_high), int(c.max_attempts),
                          int(c.topology_retries), int(c.batch), float(c.negative_rate),
                          int(self.threads or len(os.sched_getaffinity(0))), 0)

    def _run_block(self, slot0: int, nslots: int):
        torch = N.require_cuda()
        lib = N.load()
        c = self.config
        dev = self.device or torch.device("cuda")
        # two engines over the two halves of the slot range, ping-ponged on
        # two streams: one lane's host walk + window layout overlaps the
        # other lane's gate launch (results identical: slots are independent
        # and are concatenated in slot order)
        nl = 2 if (self.overlap and nslots >= 2) else 1
        cuts = [slot0 + (nslots * k) // nl for k in range(nl + 1)]
        t_init = time.perf_counter()
        lanes = [_EngineLane(self, lib, torch, dev, cuts[k], cuts[k + 1] - cuts[k], k) for k in range(nl)]
        self.timings["init"] = self.timings.get("init", 0.0) + time.perf_counter() - t_init
        try:
            for ln in lanes:
                ln.submit()
            while any(ln.active for ln in lanes):
                for ln in lanes:
                    if ln.active:
                        ln.wait_and_consume()
                        ln.submit()
            t3 = time.perf_counter()
            parts = [ln.results() for ln in lanes]
        finally:
            for ln in lanes:
                ln.close()
        meta = np.concatenate([p_[0] for p_ in parts])
        rpos = np.concatenate([p_[1] for p_ in parts])
        rplans = np.concatenate([p_[2] for p_ in parts])
        radj = np.concatenate([p_[3] for p_ in parts])
        rtypes = np.concatenate([p_[4] for p_ in parts])
        nmeta = np.concatenate([p_[5] for p_ in parts])
        npos = np.concatenate([p_[6] for p_ in parts])
        nadj = np.concatenate([p_[7] for p_ in parts])
        ntypes = np.concatenate([p_[8] for p_ in parts])
        by_n = sum(p_[9] for p_ in parts)
        disc = C.c_int64(sum(p_[10] for p_ in parts))
        R = len(meta)
        st = GenerationStats()
        for n in range(NMAX + 1):
            if by_n[n, 0] or by_n[n, 1]:
                st.simulated_by_n[n] = int(by_n[n, 0])
                st.accepted_by_n[n] = int(by_n[n, 1])
        for i in range(R):
            st.attempts_samples.setdefault(int(meta[i, 3]), []).append(int(meta[i, 2]))
        st.topologies_discarded = int(disc.value)
        negs = [NegativeSample(m, int(s)) for m, s in
                zip(_mechanisms(nadj, ntypes, npos, nmeta[:, 2]), nmeta[:, 1])]
        # T_high trajectories of the accepted variants (f64, n rows per
        # record packed back to back), one launch, one D2H
        ns = meta[:, 3].astype(np.int64)
        row0 = np.zeros(R + 1, dtype=np.int64)
        np.cumsum(ns, out=row0[1:])
        traj = np.zeros((0, c.T_high, 2))
        if R:
            table = PlanTable.from_records(rplans.reshape(-1), ns.astype(np.int32), device=dev)
            pd = torch.from_numpy(rpos[:, :int(ns.max())].copy()).to(dev)
            topo = torch.arange(R, dtype=torch.int32, device=dev)
            tbuf = torch.empty((int(row0[-1]), c.T_high, 2), dtype=torch.float64, device=dev)
            res = simulate_tensors(pd, table, c.T_high, topo, write_traj=True, traj=tbuf,
                                   traj_row=torch.from_numpy(row0[:-1]).to(dev), traj_f64=True)
            if not bool((res["first_t"] == c.T_high).all()):
                raise GenerationError("accepted variant locks at T_high on replay")
            traj = tbuf if self.traj_on_device else tbuf.cpu().numpy()
        self.timings["finish"] += time.perf_counter() - t3
        return GeneratedBlock(meta, rpos, radj, rtypes, traj, row0), st, negs

    def blocks(self):
        """Bulk output: one ``GeneratedBlock`` of arrays per slot block (all
        records of those slots, before the ``count`` cut)."""
        c = self.config
        lo, hi = self.slot_range or (0, (c.count + c.variants_per_topology - 1) // c.variants_per_topology)
        for s0 in range(lo, hi, self.slot_block):
            blk, st, negs = self._run_block(s0, min(self.slot_block, hi - s0))
            self.stats.merge(st)
            self.negatives.extend(negs)
            yield blk

    def records(self):
        """generator.py:346-375: GeneratedRecord per accepted variant, slot
        order, cut at ``count``."""
        emitted = 0
        for blk in self.blocks():
            for i in range(blk.R):
                if emitted >= self.config.count:
                    return
                emitted += 1
                yield blk.record(i)


def rejection_curve(config: GenerationConfig, sizes: list[int], trials: int = 100) -> GenerationStats:
    """Attempts-per-success study (generator.py:385-413): per joint count n,
    `trials` fresh topologies from default_rng([seed, 7_000_000 + n, 0]),
    each searched once for a valid pose on the shared stream
    default_rng([seed, 7_000_000 + n, 1]) with the GPU gate."""
    stats = GenerationStats()
    for n in sizes:
        rng_topo = np.random.default_rng([config.seed, 7_000_000 + n, 0])
        rng_pos = np.random.default_rng([config.seed, 7_000_000 + n, 1])
        for _ in range(trials):
            topology, plan = sample_topology(rng_topo, n, config.ng_probability, config.topology_retries)
            res = find_valid_variant(topology, plan, rng_pos, max_attempts=config.max_attempts,
                                     T_low=config.T_low, T_high=config.T_high, batch=config.batch)
            if res is None:
                stats.record_failure(n, config.max_attempts)
            else:
                stats.record_success(n, res.attempts)
    return stats


def generate_dataset(config: GenerationConfig, **kw):
    """generator.py:378-383: (record iterator, run object)."""
    run = GenerationRun(config, **kw)
    return run.records(), run
