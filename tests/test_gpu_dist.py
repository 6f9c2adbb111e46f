"""GPU tests of the multi-GPU retrieval path: database
shards scanned in global scan order, per-shard lists merged on the device
by la_merge_shard_lists, must equal one scan over everything; and the
torchrun launch itself (2 ranks sharing the one GPU, gloo exchange --
their kernels never wait on one another)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_scan_device_merge_equals_single_scan(torch, world):
    """world contiguous record shards, each scanned with its local order and
    global scan positions (multi-query pruned kernel, hits, an excluded
    record), packed like dist.gather_lists and merged on the device."""
    from paper_2208_14567_b200.atlas import chamfer_scan
    from paper_2208_14567_b200.dist import local_scan_plan, merge_gathered, pack_lists
    from paper_2208_14567_b200.workloads import fourier_db

    N, P, K = 240_000, 200, 8
    db = fourier_db(N, P, seed=51, chunk=1 << 16)
    q = fourier_db(12, P, seed=52)
    order = np.random.default_rng(53).permutation(N)
    dorder = torch.from_numpy(order).cuda()
    kw = dict(k=K, threshold=0.065, exclude_id=int(order[17]))
    full = chamfer_scan(db, q, order=dorder, **kw)
    assert int(full["n_hits"].sum()) > 0
    parts = []
    for r in range(world):
        lo, hi = N * r // world, N * (r + 1) // world
        lorder, pmap = local_scan_plan(order, lo, hi)
        ex = kw["exclude_id"] - lo if lo <= kw["exclude_id"] < hi else -1
        parts.append(chamfer_scan(db[lo:hi], q, k=K, threshold=kw["threshold"], exclude_id=ex,
                                  order=torch.from_numpy(lorder).cuda(), pos_map=torch.from_numpy(pmap).cuda(),
                                  id_base=lo))
    merged = merge_gathered(torch.stack([pack_lists(p, K) for p in parts]), K)
    for name in ("top_d", "top_id", "top_pos", "hit_d", "hit_id", "hit_pos", "n_hits"):
        assert torch.equal(merged[name], full[name]), name


def test_merge_kernel_matches_oracle_merge(torch):
    """la_merge_shard_lists vs the oracle's merge on random shard lists with
    empty slots, equal distances (ties broken by scan position) and hits."""
    from oracle import links_oracle as O
    from paper_2208_14567_b200.dist import merge_gathered, pack_lists

    rng = np.random.default_rng(7)
    world, NQ, K = 5, 9, 6
    parts = []
    for _ in range(world):
        p = {}
        for kind in ("top", "hit"):
            d = np.round(rng.uniform(0, 1, size=(NQ, K)), 2).astype(np.float32)  # many ties
            pos = rng.choice(1 << 40, size=(NQ, K), replace=False).astype(np.int64)
            ids = rng.integers(0, 1 << 40, size=(NQ, K)).astype(np.int64)
            empty = rng.uniform(size=(NQ, K)) < 0.3
            d[empty], pos[empty], ids[empty] = np.inf, -1, -1
            p[f"{kind}_d"], p[f"{kind}_id"], p[f"{kind}_pos"] = d, ids, pos
        p["n_hits"] = rng.integers(0, 50, size=NQ).astype(np.int64)
        parts.append(p)
    want = O.merge_shard_lists(parts, K)
    g = torch.stack([pack_lists({n: torch.from_numpy(v).cuda() for n, v in p.items()}, K) for p in parts])
    got = merge_gathered(g, K)
    for name, v in want.items():
        assert np.array_equal(got[name].cpu().numpy(), v), name


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_torchrun_two_ranks_shared_gpu():
    """torchrun --nproc-per-node 2 on the one GPU (LA_BENCH_SHARED_GPU=1,
    gloo): the launched ranks' merged lists equal the single scan."""
    env = dict(os.environ, LA_BENCH_SHARED_GPU="1", LA_DIST_N="200000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "tools", "dist_check.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    res = json.loads(line)
    assert res["world"] == 2 and res["ok"], res
