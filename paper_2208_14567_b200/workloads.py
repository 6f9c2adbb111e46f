"""Seeded synthetic inputs for the BASELINE.json configurations.

C1  1,024 four-bars (topology of the reference test fixture, conftest.py:7-18)
C2  100,000 candidates of 6-8 joints, 256 per topology, topologies and poses
    from the reference generator's PCG64 streams (generator.py:286-292)
C3  validity screen: 10M candidates of 5-20 joints, 256 per topology, from
    the same reference streams, drawn by the native multi-threaded generator
    (csrc/gen.cpp reproduces numpy's SeedSequence/PCG64/Generator and the
    topology operator bit for bit; ~0.7 s for 10M on 16 host threads)
C4  random closed Fourier curves, 5 harmonics, coefficients N(0, 1/k^2),
    generated on device and normalised once by la_normalize

The paper's LINKS dataset is not available offline; these seeded inputs
stand in for it with the shapes and distributions BASELINE.json names.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2208_14567_b200 import _native as N
from paper_2208_14567_b200.generator import _sample_positions_batch, sample_topology
from paper_2208_14567_b200.mechanism import JointType, Mechanism
from paper_2208_14567_b200.solver import PlanTable, SolutionPlan, compile_order

NMAX = N.LA_MAX_JOINTS


def four_bar(ground=(0.7, 0.5), coupler=(0.6, 0.62)) -> Mechanism:
    adj = np.zeros((4, 4), dtype=np.uint8)
    for i, j in [(0, 1), (1, 3), (2, 3)]:
        adj[i, j] = adj[j, i] = 1
    types = np.array([JointType.FIXED, JointType.ACTUATED, JointType.FIXED, JointType.SIMPLE], dtype=np.int8)
    return Mechanism(adj, types, np.array([(0.5, 0.5), (0.55, 0.5), ground, coupler]))


def bare_plan(mech: Mechanism) -> SolutionPlan:
    fixed, steps = compile_order(mech.adjacency, mech.types)
    return SolutionPlan(mech.n, fixed, steps, None, None, None)


def fourbar_batch(B: int = 1024, seed: int = 0):
    """C1: poses U[0,1)^2 with pivot/tip pinned."""
    pos = np.random.default_rng(seed).uniform(size=(B, 4, 2))
    pos[:, 0] = (0.5, 0.5)
    pos[:, 1] = (0.55, 0.5)
    return bare_plan(four_bar()), pos


@dataclass
class MixedBatch:
    plans: list[SolutionPlan]
    mechs: list[Mechanism]
    pos: np.ndarray        # (B, stride, 2) f64, NaN padded
    topo: np.ndarray       # (B,) int32
    n: np.ndarray          # (B,) joints per candidate

    @property
    def B(self) -> int:
        return len(self.topo)

    def table(self) -> PlanTable:
        return PlanTable(self.plans)


def mixed_batch(count: int, n_lo: int, n_hi: int, seed: int, per_topology: int = 256,
                stride: int | None = None) -> MixedBatch:
    """C2-style candidates: group g draws n and its topology from
    default_rng([seed, g, 0]) and its poses from default_rng([seed, g, 1])
    exactly like _generate_slot (generator.py:286-292, 225-238)."""
    groups = (count + per_topology - 1) // per_topology
    plans, mechs, poses, topo, ns = [], [], [], [], []
    stride = stride or n_hi
    left = count
    for g in range(groups):
        rt = np.random.default_rng([seed, g, 0])
        rp = np.random.default_rng([seed, g, 1])
        n = int(rt.integers(n_lo, n_hi + 1))
        mech, plan = sample_topology(rt, n)
        k = min(per_topology, left)
        left -= k
        p = _sample_positions_batch(n, k, rp)
        pad = np.full((k, stride, 2), np.nan)
        pad[:, :n] = p
        plans.append(plan)
        mechs.append(mech)
        poses.append(pad)
        topo.append(np.full(k, g, dtype=np.int32))
        ns.append(np.full(k, n, dtype=np.int32))
    return MixedBatch(plans, mechs, np.concatenate(poses), np.concatenate(topo), np.concatenate(ns))


@dataclass
class NativeBatch:
    """Candidates from the native generator (csrc/gen.cpp): group g of
    ``per_topology`` candidates uses the reference streams
    default_rng([seed, g, 0]) (n and topology) and default_rng([seed, g, 1])
    (poses), exactly like ``mixed_batch`` but for millions of candidates."""

    table: PlanTable
    types: np.ndarray      # (G, 20) int8, -1 beyond n
    n_group: np.ndarray    # (G,)
    pos: np.ndarray        # (B, stride, 2) f64
    topo: np.ndarray       # (B,) int32

    @property
    def B(self) -> int:
        return len(self.topo)


def native_batch(count: int, n_lo: int, n_hi: int, seed: int, per_topology: int = 256,
                 stride: int = NMAX) -> NativeBatch:
    from paper_2208_14567_b200.generator import native_poses, native_topologies

    G = (count + per_topology - 1) // per_topology
    raw, types, _, ns = native_topologies(seed, G, n_lo, n_hi)
    pos = native_poses(seed, ns, per_topology, stride)[:count]
    topo = (np.arange(count, dtype=np.int64) // per_topology).astype(np.int32)
    return NativeBatch(PlanTable.from_records(raw, ns), types, ns, pos, topo)


def topology_pool(G: int, n_lo: int, n_hi: int, seed: int) -> tuple[list[Mechanism], list[SolutionPlan]]:
    """G generator topologies, group g from default_rng([seed, g, 0])."""
    mechs, plans = [], []
    for g in range(G):
        rt = np.random.default_rng([seed, g, 0])
        n = int(rt.integers(n_lo, n_hi + 1))
        m, p = sample_topology(rt, n)
        mechs.append(m)
        plans.append(p)
    return mechs, plans


def device_poses(topo, plans: list[SolutionPlan], stride: int, seed: int, device=None):
    """Candidate poses drawn on device: U[0,1)^2 per joint (Philox), pivot
    and crank tip pinned (generator.py:234-238), NaN beyond each n."""
    torch = N.require_cuda()
    dev = device or torch.device("cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed))
    B = topo.numel()
    pos = torch.rand((B, stride, 2), generator=gen, dtype=torch.float64, device=dev)
    pos[:, 0, 0] = 0.5
    pos[:, 0, 1] = 0.5
    pos[:, 1, 0] = 0.55
    pos[:, 1, 1] = 0.5
    ns = torch.tensor([p.n for p in plans], dtype=torch.int64, device=dev)[topo.long()]
    j = torch.arange(stride, device=dev)[None, :]
    pos[(j >= ns[:, None])] = float("nan")
    return pos


def fourier_curves_device(count: int, P: int, seed: int, device=None, dtype=None):
    """Raw closed Fourier curves (count, P, 2): x(t) = sum_k a_k cos kt +
    b_k sin kt (same for y), k = 1..5, coefficients N(0, 1/k^2)."""
    torch = N.require_cuda()
    dev = device or torch.device("cuda")
    dt = dtype or torch.float64
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed))
    k = torch.arange(1, 6, device=dev, dtype=dt)
    coef = torch.randn((count, 4, 5), generator=gen, device=dev, dtype=dt) / k
    t = 2.0 * np.pi * torch.arange(P, device=dev, dtype=dt) / P
    ckt = torch.cos(t[:, None] * k[None, :])  # (P, 5)
    skt = torch.sin(t[:, None] * k[None, :])
    x = coef[:, 0] @ ckt.T + coef[:, 1] @ skt.T
    y = coef[:, 2] @ ckt.T + coef[:, 3] @ skt.T
    return torch.stack([x, y], dim=-1)


def fourier_db(count: int, P: int, seed: int, chunk: int = 1 << 20, device=None):
    """C4 database: Fourier curves normalised by la_normalize (f64 in,
    fp32 stored).  Returns (count, P, 2) float32 on device."""
    torch = N.require_cuda()
    from paper_2208_14567_b200.curves import normalize_tensors

    dev = device or torch.device("cuda")
    out = torch.empty((count, P, 2), dtype=torch.float32, device=dev)
    for c0 in range(0, count, chunk):
        c1 = min(count, c0 + chunk)
        raw = fourier_curves_device(c1 - c0, P, seed * 1000003 + c0 // chunk, device=dev)
        res = normalize_tensors(raw, out_f64=False)
        out[c0:c1] = res["out"]
        del raw, res
    return out
