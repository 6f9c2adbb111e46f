"""Host-side logic of the product package, checked on CPU against fixtures
the reference produced (no GPU needed)."""

import ctypes

import numpy as np
import pytest

from oracle import links_oracle as O
from paper_2208_14567_b200 import _native as N
from paper_2208_14567_b200.atlas import _content_hash, assemble_hits
from paper_2208_14567_b200.generator import GenerationConfig, GenerationStats, _sample_positions_batch, \
    sample_topology
from paper_2208_14567_b200.mechanism import JointType, Mechanism, apply_Ng, apply_Ns, compute_mobility, \
    initial_mechanism, validate
from paper_2208_14567_b200.solver import PlanError, PlanTable, SolutionPlan, compile_order
from paper_2208_14567_b200.workloads import bare_plan, four_bar


def test_compile_order_matches_reference_plans(golden):
    g = golden("solver_golden.npz")
    for t in range(len(g["mx_n"])):
        n = int(g["mx_n"][t])
        fixed, steps = compile_order(g["mx_adj"][t][:n, :n], g["mx_types"][t][:n])
        want = [tuple(int(v) for v in g["mx_steps"][t][s]) for s in range(int(g["mx_nsteps"][t]))]
        assert [(s.target, s.a, s.b) for s in steps] == want
        assert fixed == tuple(np.flatnonzero(g["mx_types"][t][:n] == 0).tolist())


def test_compile_order_unsolvable():
    adj = np.zeros((4, 4), dtype=np.uint8)
    adj[0, 1] = adj[1, 0] = 1
    adj[1, 3] = adj[3, 1] = 1
    with pytest.raises(PlanError):
        compile_order(adj, np.array([0, 2, 0, 1]))


def test_sample_topology_reproduces_reference_streams(golden):
    """Same PCG64 stream -> same topology, plan and candidate poses."""
    g = golden("solver_golden.npz")
    t = 0
    for n in [5, 6, 7, 8, 10, 12, 14, 16, 18, 20]:
        for rep in range(3):
            mech, plan = sample_topology(np.random.default_rng([7, n, rep, 0]), n)
            assert np.array_equal(mech.adjacency, g["mx_adj"][t][:n, :n])
            assert np.array_equal(mech.types, g["mx_types"][t][:n])
            assert len(plan.steps) == int(g["mx_nsteps"][t])
            pos = _sample_positions_batch(n, 64, np.random.default_rng([7, n, rep, 1]))
            assert np.array_equal(pos, g["mx_pos0"][g["mx_topo"] == t][:, :n])
            assert compute_mobility(mech).m == 1
            t += 1


def test_mechanism_operators():
    m = initial_mechanism()
    assert m.n == 3 and m.fixed_joints() == [0, 2]
    m = apply_Ns(m, 1, 2)
    assert m.types[3] == JointType.SIMPLE and compute_mobility(m).m == 1
    m = apply_Ng(m)
    assert m.types[4] == JointType.FIXED
    fb = four_bar()
    assert validate(fb) == []
    bad = Mechanism(fb.adjacency, np.array([1, 2, 0, 1]), fb.positions0)
    assert "joint 0 must be fixed" in validate(bad)
    with pytest.raises(Exception):
        apply_Ns(initial_mechanism(), 0, 2)


def test_plan_table_packing():
    plan = bare_plan(four_bar())
    raw = PlanTable([plan, plan]).host_bytes()
    assert raw.size == 128
    rec = N.LaPlan.from_buffer_copy(raw[:64].tobytes())
    assert rec.n == 4 and rec.nsteps == 1 and rec.fixed_mask == 0b101
    assert (rec.step[0][0], rec.step[0][1], rec.step[0][2]) == (3, 1, 2)
    with pytest.raises(ValueError):
        PlanTable([SolutionPlan(21, (0,), (), None, None, None)]).host_bytes()


def test_generation_config_and_stats():
    with pytest.raises(ValueError):
        GenerationConfig(count=1, n_min=3)
    with pytest.raises(ValueError):
        GenerationConfig(count=1, T_low=200, T_high=50)
    a = GenerationStats()
    a.record_success(8, 10)
    a.record_success(8, 30)
    b = GenerationStats()
    b.record_failure(8, 100)
    b.record_success(10, 7)
    a.merge(b)
    assert a.simulated_by_n[8] == 140 and a.mean_attempts(8) == 70.0 and a.median_attempts(8) == 20.0


def test_assemble_hits_matches_oracle_retrieve(golden):
    """The host half of retrieve(): device lists -> ordered hits.  Lists are
    built here from oracle distances the way the kernel defines them."""
    g = golden("atlas_golden.npz")
    pts, order = g["points"], g["order"]
    pos_of = np.empty_like(order)
    pos_of[order] = np.arange(len(order))
    for qi in range(4):
        q = g[f"query{qi}"]
        d = O.chamfer_expansion_block(pts, q)
        self_idx = None
        for i in range(len(pts)):
            if pts[i].shape == q.shape and pts[i].tobytes() == q.tobytes():
                self_idx = i
        for k, thr in zip(g["cases_k"], g["cases_thr"]):
            k = int(k)
            keep = np.array([i for i in range(len(pts)) if i != self_idx])
            hit = keep[d[keep] < thr]
            hit = hit[np.argsort(pos_of[hit], kind="stable")][:k]
            non = keep[d[keep] >= thr]
            non = non[np.lexsort((pos_of[non], d[non]))][:k]
            got = assemble_hits(d[hit], hit, d[non], non, k, thr, self_idx)
            want = O.retrieve(pts, order, q, k, thr)
            assert [r[1] for r in got] == [r[1] for r in want]
            assert [r[2] for r in got] == [bool(r[2]) for r in want]


def test_content_hash_distinguishes_records(golden):
    g = golden("atlas_golden.npz")
    h = _content_hash(g["points"])
    assert len(np.unique(h)) == len(h)
    assert _content_hash(g["points"][17:18])[0] == h[17]


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the ABI structs have the C layout (gcc here)."""
    import subprocess

    from conftest import ROOT

    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "links_b200.h"\n'
        "int main(){printf(\"%zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(la_plan), sizeof(la_sim_args),"
        " sizeof(la_norm_args), sizeof(la_chamfer_args), offsetof(la_sim_args, fixup_tau),"
        " offsetof(la_chamfer_args, ws_bytes), offsetof(la_norm_args, rel_tol));return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", f"{ROOT}/include", str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(N.LaPlan), ctypes.sizeof(N.LaSimArgs), ctypes.sizeof(N.LaNormArgs),
            ctypes.sizeof(N.LaChamferArgs), N.LaSimArgs.fixup_tau.offset, N.LaChamferArgs.ws_bytes.offset,
            N.LaNormArgs.rel_tol.offset]
    assert got == want


def test_sample_topology_leaves_reference_stream_state(golden):
    """Two topologies in sequence from one Generator, then the next draws:
    the native operator advances the caller's PCG64 state exactly as the
    reference's draws do (generator.py:200-222)."""
    g = golden("stream_golden.npz")
    for c in range(len(g["n"])):
        rng = np.random.default_rng([99, c])
        n = int(rng.integers(5, 21))
        assert n == int(g["n"][c])
        for k in range(2):
            mech, _ = sample_topology(rng, n)
            assert np.array_equal(mech.adjacency, g["adj"][c, k][:n, :n])
            assert np.array_equal(mech.types, g["types"][c, k][:n])
        assert np.array_equal(rng.random(2), g["after"][c, :2])
        assert int(rng.integers(1000)) == int(g["after"][c, 2])
