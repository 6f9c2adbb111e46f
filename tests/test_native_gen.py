"""The native generator (csrc/gen.cpp) reproduces numpy's PCG64 streams and
the reference topology operator bit for bit (CPU only)."""

import ctypes

import numpy as np
import pytest

from paper_2208_14567_b200 import _native as N
from paper_2208_14567_b200.generator import _sample_positions_batch, native_poses, native_topologies, \
    sample_topology
from paper_2208_14567_b200.solver import PlanTable


@pytest.mark.parametrize("ent", [[0], [7], [7, 5, 0], [2208, 390, 1], [2**33 + 5, 0, 2], [123456789, 99999, 1]])
def test_pcg64_streams_match_numpy(ent):
    lib = N.load()
    e = np.array(ent, dtype=np.int64)
    d = np.empty(1000)
    lib.la_rng_draw(e.ctypes.data, len(ent), 0, 0, 1000, d.ctypes.data, None)
    assert np.array_equal(d, np.random.default_rng(ent).random(1000))
    for bound in (1, 2, 3, 7, 100, 1000, 2**31 - 1):
        got = np.empty(500, dtype=np.int64)
        lib.la_rng_draw(e.ctypes.data, len(ent), 1, bound, 500, None, got.ctypes.data)
        rng = np.random.default_rng(ent)
        want = np.array([rng.integers(bound) for _ in range(500)])
        assert np.array_equal(got, want), bound


def test_topologies_match_reference_operator():
    seed, G = 11, 60
    plans, types, adj, ns = native_topologies(seed, G, 5, 20)
    for g in range(G):
        rt = np.random.default_rng([seed, g, 0])
        n = int(rt.integers(5, 21))
        mech, plan = sample_topology(rt, n)
        assert ns[g] == n
        assert np.array_equal(adj[g][:n, :n], mech.adjacency)
        assert np.array_equal(types[g][:n], mech.types)
        assert plans[g * 64:(g + 1) * 64].tobytes() == PlanTable([plan]).host_bytes().tobytes()


def test_poses_match_reference_sampler():
    ns = np.array([6, 8, 20, 5], dtype=np.int32)
    pos = native_poses(3, ns, 37, 20, g0=100)
    for g, n in enumerate(ns):
        want = _sample_positions_batch(int(n), 37, np.random.default_rng([3, 100 + g, 1]))
        got = pos[g * 37:(g + 1) * 37]
        assert np.array_equal(got[:, :n], want)
        assert np.isnan(got[:, n:]).all()


def test_native_batch_equals_mixed_batch():
    from paper_2208_14567_b200.workloads import mixed_batch, native_batch

    a = mixed_batch(1000, 6, 8, seed=5, stride=8)
    b = native_batch(1000, 6, 8, seed=5, stride=8)
    assert np.array_equal(a.topo, b.topo)
    assert np.array_equal(a.pos, b.pos, equal_nan=True)
    assert a.table().host_bytes().tobytes() == b.table.host_bytes().tobytes()
