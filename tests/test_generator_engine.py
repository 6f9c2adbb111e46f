"""Host logic of the dataset-generation engine (la_gen_*) against the
reference GenerationRun fixtures, with the ORACLE answering the two-fidelity
gate on CPU (the GPU answers it in tests/test_gpu_generator.py).  The engine
must reproduce records (slot, variant, attempts, poses), negatives and stats
bit for bit — only the gate evaluation differs between the two tests."""

import ctypes as C

import numpy as np
import pytest

from oracle import links_oracle as O
from paper_2208_14567_b200 import _native as N

NMAX = N.LA_MAX_JOINTS


def _cfg(g, ci):
    cfg = g[f"g{ci}_cfg"]
    rates = g[f"g{ci}_rates"]
    count, seed, n_min, n_max, vpt, T_low, T_high, max_att, batch, retries = (int(x) for x in cfg)
    return count, N.LaGenCfg(seed, n_min, n_max, float(rates[0]), vpt, T_low, T_high, max_att, retries, batch,
                             float(rates[1]), 4, 0)  # 4 host threads: parallel flag walks


def _oracle_gate(pos, cand_plan, plans, m, T_low, T_high):
    """first_t at T_high and the T_low lock step (-1 if none) per candidate."""
    first = np.empty(m, dtype=np.int32)
    low = np.empty(m, dtype=np.int32)
    for p in np.unique(cand_plan[:m]):
        rec = plans[p]
        n = int(rec.n)
        steps = [tuple(int(v) for v in rec.step[s]) for s in range(rec.nsteps)]
        fixed = [k for k in range(n) if (rec.fixed_mask >> k) & 1]
        idx = np.nonzero(cand_plan[:m] == p)[0]
        x = pos[idx, :n]
        lo = O.simulate(x, steps, fixed, T_low)["first_t"]
        hi = O.simulate(x, steps, fixed, T_high)["first_t"]
        low[idx] = np.where(lo < T_low, lo, -1)
        first[idx] = hi
    return first, low


def _numpy_poses(batches, nb, m):
    """Poses of a device-drawn window, drawn by numpy from the descriptors."""
    pos = np.full((m, NMAX, 2), np.nan)
    cand_plan = np.zeros(m, dtype=np.int32)
    bg = np.random.PCG64()
    for i in range(nb):
        b = batches[i]
        bg.state = {"bit_generator": "PCG64",
                    "state": {"state": (b.state_hi << 64) | b.state_lo, "inc": (b.inc_hi << 64) | b.inc_lo},
                    "has_uint32": 0, "uinteger": 0}
        x = np.random.Generator(bg).uniform(size=(b.k, b.n, 2))
        x[:, 0] = (0.5, 0.5)
        x[:, 1] = (0.55, 0.5)
        pos[b.first:b.first + b.k, :b.n] = x
        cand_plan[b.first:b.first + b.k] = b.plan
    return pos, cand_plan


def run_engine(cfg, count, lookahead=3, cap=1 << 16, device_windows=False, slot0=0, nslots=None):
    lib = N.load()
    slots = (count + cfg.variants - 1) // cfg.variants if nslots is None else nslots
    eng = lib.la_gen_create(C.byref(cfg), slot0, slots)
    assert eng
    try:
        pos = np.zeros((cap, NMAX, 2))
        cand_plan = np.zeros(cap, dtype=np.int32)
        plans = (N.LaPlan * slots)()
        n_plans = C.c_int32(0)
        batches = (N.LaGenBatch * 4096)()
        nb = C.c_int64(0)
        windows = 0
        while True:
            if device_windows:
                m = lib.la_gen_window_dev(eng, lookahead, cap, batches, 4096, C.byref(nb), plans, C.byref(n_plans))
            else:
                m = lib.la_gen_window(eng, lookahead, cap, 2, pos.ctypes.data, cand_plan.ctypes.data, plans,
                                      C.byref(n_plans))
            assert m >= 0, N.last_error()
            if m == 0:
                break
            windows += 1
            if device_windows:
                pos, cand_plan = _numpy_poses(batches, nb.value, m)
            first, low = _oracle_gate(pos, cand_plan, plans, m, cfg.T_low, cfg.T_high)
            src = None if device_windows else pos.ctypes.data
            assert lib.la_gen_consume(eng, src, first.ctypes.data, low.ctypes.data) == 0
        R = lib.la_gen_count(eng, 0)
        meta = np.zeros((R, 4), dtype=np.int64)
        rpos = np.zeros((R, NMAX, 2))
        rplans = (N.LaPlan * max(R, 1))()
        adj = np.zeros((R, NMAX, NMAX), dtype=np.uint8)
        types = np.zeros((R, NMAX), dtype=np.int8)
        assert lib.la_gen_records(eng, meta.ctypes.data, rpos.ctypes.data, rplans, adj.ctypes.data,
                                  types.ctypes.data) == 0
        Q = lib.la_gen_count(eng, 1)
        nmeta = np.zeros((Q, 3), dtype=np.int64)
        npos = np.zeros((Q, NMAX, 2))
        assert lib.la_gen_negatives(eng, nmeta.ctypes.data, npos.ctypes.data,
                                    np.zeros((Q, NMAX, NMAX), dtype=np.uint8).ctypes.data,
                                    np.zeros((Q, NMAX), dtype=np.int8).ctypes.data) == 0
        by_n = np.zeros((NMAX + 1, 2), dtype=np.int64)
        disc = C.c_int64(0)
        assert lib.la_gen_stats(eng, by_n.ctypes.data, C.byref(disc)) == 0
    finally:
        lib.la_gen_destroy(eng)
    return dict(meta=meta, pos=rpos, adj=adj, types=types, nmeta=nmeta, npos=npos, by_n=by_n, disc=disc.value,
                windows=windows)


def check_against_golden(g, ci, out, count):
    meta = out["meta"][:count]
    assert np.array_equal(meta, g[f"g{ci}_meta"])
    want_pos = g[f"g{ci}_pos"]
    for i, n in enumerate(meta[:, 3]):
        assert np.array_equal(out["pos"][i, :n], want_pos[i, :n])
        assert np.array_equal(out["adj"][i, :n, :n], g[f"g{ci}_adj"][i, :n, :n])
    stats = g[f"g{ci}_stats"]
    got = np.array([[n, out["by_n"][n, 0], out["by_n"][n, 1]] for n in stats[:, 0]])
    assert np.array_equal(got, stats)
    assert int(out["by_n"][:, 0].sum()) == int(stats[:, 1].sum())
    assert out["disc"] == int(g[f"g{ci}_discarded"])
    negstep = g[f"g{ci}_negstep"]
    assert np.array_equal(out["nmeta"][:, 1], negstep)
    for i, n in enumerate(out["nmeta"][:, 2]):
        assert np.array_equal(out["npos"][i, :n], g[f"g{ci}_neg"][i, :n])


@pytest.mark.parametrize("ci", [0, 1, 2])
def test_engine_matches_reference_run(golden, ci):
    g = golden("generator_golden.npz")
    count, cfg = _cfg(g, ci)
    out = run_engine(cfg, count)
    check_against_golden(g, ci, out, count)


@pytest.mark.parametrize("ci", [1, 2])
def test_engine_device_windows(golden, ci):
    """Descriptor windows (stream states jumped ahead on the host, poses of
    accepted / negative candidates redrawn from them) give the same run."""
    g = golden("generator_golden.npz")
    count, cfg = _cfg(g, ci)
    out = run_engine(cfg, count, lookahead=5, device_windows=True)
    check_against_golden(g, ci, out, count)


def test_engine_lookahead_invariance(golden):
    """Look-ahead depth and window cap change only how much is screened."""
    g = golden("generator_golden.npz")
    count, cfg = _cfg(g, 2)
    a = run_engine(cfg, count, lookahead=1)
    b = run_engine(cfg, count, lookahead=7, cap=2048)
    for k in ("meta", "pos", "nmeta", "npos", "by_n"):
        assert np.array_equal(a[k], b[k], equal_nan=True)
    assert a["windows"] >= 2 and b["windows"] >= 2


def test_engine_slot_shards_concatenate(golden):
    """Rank r of N owns a contiguous slot range (bench.py / GenerationRun
    slot_range): shards generate independently and concatenate to the
    single-engine run, stats summing -- no collective needed."""
    g = golden("generator_golden.npz")
    count, cfg = _cfg(g, 2)
    slots = (count + cfg.variants - 1) // cfg.variants
    whole = run_engine(cfg, count)
    half = slots // 2
    a = run_engine(cfg, count, slot0=0, nslots=half)
    b = run_engine(cfg, count, slot0=half, nslots=slots - half)
    assert np.array_equal(np.concatenate([a["meta"], b["meta"]]), whole["meta"])
    assert np.array_equal(np.concatenate([a["pos"], b["pos"]]), whole["pos"], equal_nan=True)
    assert np.array_equal(a["by_n"] + b["by_n"], whole["by_n"])
    assert a["disc"] + b["disc"] == whole["disc"]


def test_engine_bad_config():
    lib = N.load()
    cfg = N.LaGenCfg(0, 3, 8, 0.25, 5, 50, 200, 5000, 1000, 256, 0.0)
    assert not lib.la_gen_create(C.byref(cfg), 0, 4)
    cfg = N.LaGenCfg(0, 20, 20, 0.25, 5, 50, 200, 5000, 1000, 256, 0.0)
    eng = lib.la_gen_create(C.byref(cfg), 0, 0)
    assert eng
    n_plans = C.c_int32(0)
    assert lib.la_gen_window(eng, 2, 16, 1, None, None, None, C.byref(n_plans)) == 0
    lib.la_gen_destroy(eng)


def test_moving_joint_rows_follow_cli_normalize(golden):
    """dataset.moving_joint_rows enumerates curves like cli.normalize
    (cli.py:124-136): records in order, non-Fixed joints ascending, mech id
    slot * variants + variant, is_arc = any Fixed neighbour (curves.py:87-92);
    rows index the packed trajectory block."""
    from paper_2208_14567_b200.dataset import moving_joint_rows
    from paper_2208_14567_b200.generator import GeneratedBlock

    g = golden("generator_golden.npz")
    count, cfg = _cfg(g, 0)
    out = run_engine(cfg, count)
    meta, adj, types = out["meta"], out["adj"], out["types"]
    ns = meta[:, 3]
    row0 = np.zeros(len(ns) + 1, dtype=np.int64)
    np.cumsum(ns, out=row0[1:])
    blk = GeneratedBlock(meta, out["pos"], adj, types, np.zeros((0, 1, 2)), row0)
    rows, mids, jids, arc = moving_joint_rows(blk, cfg.variants)
    want = []
    for i in range(len(meta)):
        n = int(ns[i])
        for j in range(n):
            if types[i, j] == 0:
                continue
            nbrs = np.flatnonzero(adj[i, j, :n])
            want.append((row0[i] + j, meta[i, 0] * cfg.variants + meta[i, 1], j, bool((types[i, nbrs] == 0).any())))
    got = list(zip(rows.tolist(), mids.tolist(), jids.tolist(), arc.tolist()))
    assert got == [tuple(int(x) if k < 3 else x for k, x in enumerate(w)) for w in want]


def test_engine_infeasible_size_raises():
    """n = 4 has no valid topology (SURVEY probe P0): the reference raises
    GenerationError from sample_topology; the engine reports LA_ERANGE with
    the same message shape on its first window."""
    lib = N.load()
    cfg = N.LaGenCfg(0, 4, 4, 0.25, 5, 50, 200, 5000, 50, 256, 0.0, 1, 0)
    eng = lib.la_gen_create(C.byref(cfg), 0, 2)
    assert eng
    n_plans = C.c_int32(0)
    pos = np.zeros((1024, NMAX, 2))
    plan = np.zeros(1024, dtype=np.int32)
    plans = (N.LaPlan * 2)()
    rc = lib.la_gen_window(eng, 1, 1024, 1, pos.ctypes.data, plan.ctypes.data, plans, C.byref(n_plans))
    assert rc == N.LA_ERANGE
    assert "no valid topology with n=4" in N.last_error()
    lib.la_gen_destroy(eng)
