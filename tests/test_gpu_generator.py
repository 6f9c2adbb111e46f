"""GenerationRun on the GPU gate vs the reference GenerationRun fixtures:
records (slot, variant, attempts, poses, topology), T_high trajectories,
negatives and stats.  Poses and attempts are bit-exact; trajectories within
1e-9 (f64 write path; the fixture holds the last joint's T_high path)."""

import numpy as np
import pytest

from paper_2208_14567_b200.generator import GenerationConfig, GenerationRun, generate_dataset

pytestmark = pytest.mark.gpu


def _config(g, ci):
    count, seed, n_min, n_max, vpt, T_low, T_high, max_att, batch, retries = (int(x) for x in g[f"g{ci}_cfg"])
    ng, neg = (float(x) for x in g[f"g{ci}_rates"])
    return GenerationConfig(count=count, n_min=n_min, n_max=n_max, ng_probability=ng, variants_per_topology=vpt,
                            T_low=T_low, T_high=T_high, max_attempts=max_att, seed=seed, negative_rate=neg,
                            topology_retries=retries, batch=batch)


@pytest.mark.parametrize("ci", [0, 1, 2])
def test_generation_run_matches_reference(golden, ci):
    g = golden("generator_golden.npz")
    cfg = _config(g, ci)
    run = GenerationRun(cfg, lookahead=3)
    recs = list(run.records())
    meta = g[f"g{ci}_meta"]
    assert len(recs) == len(meta)
    for r, m, p, adj, last in zip(recs, meta, g[f"g{ci}_pos"], g[f"g{ci}_adj"], g[f"g{ci}_traj_last"]):
        n = int(m[3])
        assert (r.slot, r.variant, r.attempts, r.mechanism.n) == tuple(int(x) for x in m)
        assert np.array_equal(r.mechanism.positions0, p[:n])
        assert np.array_equal(r.mechanism.adjacency, adj[:n, :n])
        assert r.trajectory.positions.shape == (n, cfg.T_high, 2)
        assert np.max(np.abs(r.trajectory.positions[-1] - last)) <= 1e-9
    st = g[f"g{ci}_stats"]
    for n, sim, acc in st:
        assert run.stats.simulated_by_n.get(int(n), 0) == sim
        assert run.stats.accepted_by_n.get(int(n), 0) == acc
    assert run.stats.topologies_discarded == int(g[f"g{ci}_discarded"])
    negstep = g[f"g{ci}_negstep"]
    assert [x.locking_step for x in run.negatives] == list(negstep)
    for x, p in zip(run.negatives, g[f"g{ci}_neg"]):
        assert np.array_equal(x.mechanism.positions0, p[:x.mechanism.n])


def test_generation_split_gate_and_blocks(golden):
    """T_high != 4 T_low uses two launches; slot blocks and look-ahead depth
    must not change the result."""
    g = golden("generator_golden.npz")
    cfg = _config(g, 2)
    a = list(GenerationRun(cfg, lookahead=1, slot_block=3).records())
    it, run = generate_dataset(cfg, lookahead=6)
    b = list(it)
    assert [(r.slot, r.variant, r.attempts) for r in a] == [(r.slot, r.variant, r.attempts) for r in b]
    cfg2 = GenerationConfig(count=8, n_min=5, n_max=7, variants_per_topology=2, T_low=40, T_high=120, seed=3,
                            max_attempts=400)
    recs = list(GenerationRun(cfg2).records())
    assert len(recs) == 8 and all(r.trajectory.positions.shape[1] == 120 for r in recs)


def test_device_poses_bit_exact():
    """la_gen_poses draws exactly numpy's uniform(size=(k, n, 2)) from a
    jumped PCG64 state, pivot / tip pinned, NaN beyond n."""
    import ctypes as C

    import torch

    from paper_2208_14567_b200 import _native as N

    lib = N.load()
    rng = np.random.default_rng(99)
    nb = 7
    desc = (N.LaGenBatch * nb)()
    want = []
    first = 0
    for i in range(nb):
        bg = np.random.PCG64([int(x) for x in rng.integers(0, 2**31, size=3)])
        st = bg.state["state"]
        n, k = int(rng.integers(4, 21)), int(rng.integers(1, 600))
        d = desc[i]
        d.state_hi, d.state_lo = st["state"] >> 64, st["state"] & ((1 << 64) - 1)
        d.inc_hi, d.inc_lo = st["inc"] >> 64, st["inc"] & ((1 << 64) - 1)
        d.first, d.k, d.n, d.plan = first, k, n, i
        x = np.random.Generator(bg).uniform(size=(k, n, 2))
        x[:, 0] = (0.5, 0.5)
        x[:, 1] = (0.55, 0.5)
        want.append((first, k, n, x))
        first += k
    raw = np.frombuffer(bytes(desc), dtype=np.uint8)
    dd = torch.from_numpy(raw.copy()).cuda()
    pos = torch.empty((first, 20, 2), dtype=torch.float64, device="cuda")
    topo = torch.empty(first, dtype=torch.int32, device="cuda")
    N.check(lib.la_gen_poses(dd.data_ptr(), nb, 20, pos.data_ptr(), topo.data_ptr(), N.stream_ptr()), "poses")
    got = pos.cpu().numpy()
    tp = topo.cpu().numpy()
    for i, (f, k, n, x) in enumerate(want):
        assert np.array_equal(got[f:f + k, :n], x)
        assert np.isnan(got[f:f + k, n:]).all()
        assert (tp[f:f + k] == i).all()


def test_host_and_device_windows_agree(golden):
    g = golden("generator_golden.npz")
    cfg = _config(g, 1)
    a = GenerationRun(cfg, device_poses=False)
    b = GenerationRun(cfg, device_poses=True, lookahead=9)
    ra, rb = list(a.records()), list(b.records())
    assert [(r.slot, r.variant, r.attempts) for r in ra] == [(r.slot, r.variant, r.attempts) for r in rb]
    assert all(np.array_equal(x.mechanism.positions0, y.mechanism.positions0) for x, y in zip(ra, rb))
    assert [x.locking_step for x in a.negatives] == [x.locking_step for x in b.negatives]


def test_generation_error_like_reference():
    """No valid topology for n = 4 (reference: GenerationError)."""
    from paper_2208_14567_b200.generator import GenerationError

    with pytest.raises(GenerationError, match="n=4"):
        list(GenerationRun(GenerationConfig(count=2, n_min=4, n_max=4, topology_retries=20)).records())
