"""C5's chain against the oracle at a size the oracle finishes in seconds:
two-fidelity gate of 5-20 joint generator candidates -> f64 replay of the
valid ones -> fp32 normalisation of every moving-joint path (cli.py:131-134)
-> chamfer top-10 of Fourier queries (an exhaustive scan at this size; the
pruned multi-query kernel on C5's sizes is pinned to the exhaustive lists by
test_gpu_atlas.py::test_multi_query_scan_equals_unpruned).  Valid set equal to
the oracle gate outside the 1e-6 margin band; normalised coordinates within
1e-4 on frame-stable curves; listed distances within 1e-4 of the oracle's
(f64 normalisation + direct-difference chamfer) and no frame-stable curve
beating a query's k-th distance left out of its list."""

import numpy as np
import pytest

from oracle import links_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


def _plans(table):
    raw = table.host_bytes().reshape(-1, 64)
    out = []
    for r in raw:
        n = int(r[0:2].view(np.int16)[0])
        S = int(r[2:4].view(np.int16)[0])
        mask = int(r[4:8].view(np.uint32)[0])
        st = r[8:8 + 54].view(np.int8).reshape(18, 3)
        out.append((n, [(int(st[s, 0]), int(st[s, 1]), int(st[s, 2])) for s in range(S)],
                    tuple(j for j in range(n) if (mask >> j) & 1)))
    return out


def test_c5_chain_matches_oracle(torch):
    from paper_2208_14567_b200.atlas import chamfer_scan
    from paper_2208_14567_b200.curves import normalize_tensors
    from paper_2208_14567_b200.solver import compact_valid, simulate_tensors
    from paper_2208_14567_b200.workloads import fourier_db, native_batch

    nb = native_batch(7 * 256, 5, 20, seed=5077)
    plans = _plans(nb.table)
    pos, topo = torch.from_numpy(nb.pos).cuda(), torch.from_numpy(nb.topo).cuda()
    res = simulate_tensors(pos, nb.table, 200, topo, write_traj=False, gate_only=True)
    idx, cnt = compact_valid(res["first_t"], 200)
    nv = int(cnt.item())
    assert nv > 50
    traj = torch.empty((nv * 20, 200, 2), dtype=torch.float32, device="cuda")
    simulate_tensors(pos, nb.table, 200, topo, write_traj=True, traj=traj, traj_stride=20, cand=idx[:nv],
                     coarse=False)
    moving = torch.from_numpy(nb.types > 0).cuda()
    mv = moving[topo[idx[:nv]].long()]
    rows = (torch.arange(nv, device="cuda")[:, None] * 20 + torch.arange(20, device="cuda"))[mv]
    nres = normalize_tensors(traj, src_row=rows)
    q = fourier_db(4, 200, seed=5151)
    cres = chamfer_scan(nres["out"], q, k=10, threshold=0.0)

    # oracle: gate, f64 paths, f64 normalisation of the same moving joints
    valid_gpu = (res["first_t"].cpu().numpy() == 200)
    valid_ref = np.zeros(len(nb.pos), bool)
    near = np.zeros(len(nb.pos), bool)
    curves, stable = [], []
    for g in range(len(plans)):
        n, steps, fixed = plans[g]
        lo, hi = g * 256, min((g + 1) * 256, len(nb.pos))
        v, _ = O.gate(nb.pos[lo:hi, :n], steps, fixed)
        valid_ref[lo:hi] = v
        r = O.simulate(nb.pos[lo:hi, :n], steps, fixed, 200, with_margin=True)
        near[lo:hi] = r["margin"] < 1e-6
    assert not np.any((valid_gpu != valid_ref) & ~near)
    vidx = idx[:nv].cpu().numpy()
    for b in vidx:
        n, steps, fixed = plans[nb.topo[b]]
        r = O.simulate(nb.pos[b:b + 1, :n], steps, fixed, 200)
        ok_b = int(r["first_t"][0]) == 200  # a near-margin disagreement has no oracle path
        P = O.trajectories(r)[0]
        for j in range(n):
            if nb.types[nb.topo[b], j] > 0:
                curves.append(O.normalize(P[j]) if ok_b else np.full((200, 2), np.nan))
                stable.append(ok_b and O.frame_stability(P[j]))
    curves = np.stack(curves)
    stable = np.array(stable)
    assert len(curves) == rows.numel()
    out = nres["out"].cpu().numpy().astype(np.float64)
    ok = stable & ~nres["unstable"].cpu().numpy().astype(bool)
    assert ok.sum() > 0.5 * len(curves)
    assert np.max(np.abs(out[ok] - curves[ok])) <= TOL

    qs = q.cpu().numpy().astype(np.float64)
    cz = np.where(np.isnan(curves), 0.0, curves)
    for qi in range(len(qs)):
        d_ref = O.chamfer_direct_block(cz, qs[qi])
        ids = cres["top_id"][qi].cpu().numpy()
        dd = cres["top_d"][qi].cpu().numpy()
        assert np.all(np.diff(dd) >= 0)
        for i, d in zip(ids, dd):
            if stable[i]:
                assert abs(d - d_ref[i]) <= TOL, (qi, i)
        kth = dd[-1]
        listed = set(ids.tolist())
        better = np.flatnonzero(stable & (d_ref < kth - 2 * TOL))
        assert set(better.tolist()) <= listed, qi
