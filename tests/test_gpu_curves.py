"""GPU parity of normalisation, is_circle and chamfer against reference
fixtures and the oracle.  Tolerance: 1e-4 of the bounding-box diagonal for
coordinates and distances (north_star); frame-unstable curves (near-tied
farthest pair, first point on the flip boundary) are excluded and counted."""

import numpy as np
import pytest

from oracle import links_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


def test_normalize_dropin_matches_reference(torch, golden):
    from paper_2208_14567_b200 import DegeneratePathError, normalize
    from paper_2208_14567_b200.curves import is_normalized

    g = golden("curves_golden.npz")
    for p, want in zip(g["paths"], g["normalized"]):
        got = normalize(p)  # f64 kernel path
        assert np.max(np.abs(got - want)) <= 1e-9
    assert np.array_equal(normalize(np.array([[2.0, 2.0], [4.0, 2.0]])), g["two_point"])
    assert [is_normalized(x) for x in g["normalized"]] == list(g["is_normalized"])
    assert [is_normalized(x) for x in g["paths"][:12]] == list(g["is_normalized_raw"][:12])
    with pytest.raises(DegeneratePathError):
        normalize(np.full((10, 2), 0.3))
    with pytest.raises(ValueError):
        normalize(np.zeros((1, 2)))


def test_normalize_batch_fp32_vs_reference(torch, golden):
    from paper_2208_14567_b200.curves import normalize_tensors

    g = golden("curves_golden.npz")
    paths = torch.from_numpy(g["paths"].astype(np.float32)).cuda()
    res = normalize_tensors(paths)
    out = res["out"].cpu().numpy().astype(np.float64)
    pair = res["pair"].cpu().numpy()
    unstable = res["unstable"].cpu().numpy().astype(bool)
    circ = res["is_circle"].cpu().numpy().astype(bool)
    checked = 0
    for m in range(len(out)):
        stable_ref = O.frame_stability(g["paths"][m])
        # every curve stable with a 10x margin (farthest pair unique within
        # 1e-5, first point 1e-5 off the flip line) must be compared: the
        # GPU may not call it unstable
        if O.frame_stability(g["paths"][m], rel=1e-5, y_tol=1e-5):
            assert not unstable[m], m
        if unstable[m] or not stable_ref:
            continue
        checked += 1
        assert tuple(pair[m]) == tuple(g["pairs"][m])
        # normalised coordinates: unit diameter, so the diagonal is >= 1
        assert np.max(np.abs(out[m] - g["normalized"][m])) <= 1e-4
        if abs(g["circle_var"][m] - 5e-4) > 1e-6:
            assert circ[m] == g["is_circle"][m]
    assert checked >= len(out) // 2
    print(f"\nnormalize fp32: {checked}/{len(out)} frame-stable curves compared")


def test_is_circle(torch, golden):
    from paper_2208_14567_b200 import is_circle, normalize

    t = np.linspace(0, 2 * np.pi, 100, endpoint=False)
    assert is_circle(normalize(np.stack([np.cos(t), np.sin(t)], axis=1) * 3.0 + 7.0))
    r = np.full(100, 0.5)
    r[:50] += np.sqrt(5e-4)
    r[50:] -= np.sqrt(5e-4)
    synthetic = np.stack([0.5 + r * np.cos(t), 0.5 + r * np.sin(t)], axis=1)
    assert not is_circle(synthetic)  # exactly at the threshold: strict <
    g = golden("curves_golden.npz")
    for x, want in zip(g["normalized"], g["is_circle"]):
        assert is_circle(x) == bool(want)


def test_chamfer_dropin(torch, golden):
    from paper_2208_14567_b200 import chamfer

    g = golden("curves_golden.npz")
    A, B = g["normalized"][:16], g["normalized"][16:32]
    for i in range(0, 16, 3):
        for j in range(0, 16, 5):
            assert abs(chamfer(A[i], B[j]) - g["chamfer_AB"][i, j]) <= 1e-4
    assert chamfer(np.array([[0.0, 0.0]]), np.array([[1.0, 0.0]])) == 2.0
    assert chamfer(A[0], A[0]) == 0.0
    assert chamfer(A[1], B[2]) == pytest.approx(chamfer(B[2], A[1]), abs=1e-6)
    # odd point counts / Q > 256 exercise the generic kernel
    odd = A[0][:199]
    assert abs(chamfer(odd, B[0]) - O.chamfer(odd, B[0])) <= 1e-4
    big = np.concatenate([A[0], A[1]])  # 400 query points
    assert abs(chamfer(B[3], big) - O.chamfer(B[3], big)) <= 1e-4


@pytest.mark.parametrize("P,Q", [(200, 200), (64, 64), (64, 3), (200, 37), (2, 256)])
def test_chamfer_block_shapes(torch, P, Q):
    from paper_2208_14567_b200.curves import chamfer_block

    rng = np.random.default_rng(P * 1000 + Q)
    pts = rng.uniform(size=(300, P, 2))
    q = rng.uniform(size=(Q, 2))
    got = chamfer_block(torch.from_numpy(pts).cuda(), torch.from_numpy(q).cuda()).cpu().numpy()
    want = O.chamfer_direct_block(pts.astype(np.float32).astype(np.float64), q.astype(np.float32).astype(np.float64))
    assert np.max(np.abs(got - want)) <= 1e-4 * np.sqrt(2)


@pytest.mark.parametrize("P", [2, 3, 7, 63, 200, 201, 1500])
def test_normalize_sizes_f64_and_f32(torch, P):
    from paper_2208_14567_b200.curves import normalize_tensors

    rng = np.random.default_rng(P)
    t = np.linspace(0, 2 * np.pi, P, endpoint=False)
    paths = np.stack([np.stack([np.cos(t) * (1 + 0.3 * rng.random()) + 0.1 * np.cos(3 * t + rng.random()),
                                np.sin(2 * t) * 0.4 + 0.05 * rng.normal(size=P)], 1) for _ in range(4)])
    r64 = normalize_tensors(torch.from_numpy(paths).cuda())
    for m in range(4):
        want = O.normalize(paths[m])
        assert np.max(np.abs(r64["out"][m].cpu().numpy() - want)) <= 1e-9
        i, j, d = O.farthest_pair(paths[m])
        assert tuple(r64["pair"][m].tolist()) == (i, j)
        assert abs(float(r64["diameter"][m]) - d) <= 1e-12 * max(d, 1.0)
    r32 = normalize_tensors(torch.from_numpy(paths.astype(np.float32)).cuda())
    for m in range(4):
        if int(r32["unstable"][m]) == 0 and O.frame_stability(paths[m].astype(np.float32).astype(np.float64)):
            want = O.normalize(paths[m].astype(np.float32).astype(np.float64))
            assert np.max(np.abs(r32["out"][m].cpu().numpy() - want)) <= 1e-4


def test_normalize_degenerate_batch_status(torch):
    from paper_2208_14567_b200.curves import normalize_tensors

    paths = np.zeros((3, 10, 2))
    paths[1] = np.random.default_rng(0).uniform(size=(10, 2))
    res = normalize_tensors(torch.from_numpy(paths).cuda())
    assert res["status"].tolist() == [1, 0, 1]


def test_normalize_f64_bit_exact(torch, golden):
    """f64 la_normalize reproduces curves.normalize bit for bit (cdist
    without contraction, OpenBLAS's FMA order for the rotation, IEEE
    division) and np.var for is_circle (pairwise summation order)."""
    from paper_2208_14567_b200.curves import normalize_tensors

    g = golden("curves_golden.npz")
    res = normalize_tensors(torch.from_numpy(g["paths"]).cuda(), out_f64=True)
    out = res["out"].cpu().numpy()
    same = [np.array_equal(o, w) for o, w in zip(out, g["normalized"])]
    assert all(same), f"{len(same) - sum(same)} of {len(same)} curves differ"
    assert np.array_equal(res["circle_var"].cpu().numpy(), g["circle_var"])
    assert np.array_equal(res["is_circle"].cpu().numpy().astype(bool), g["is_circle"])
