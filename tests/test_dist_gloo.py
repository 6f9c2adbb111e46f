"""world_size-2 gloo test of the multi-GPU exchange path (CPU): each rank
builds its shard's (Q x k) lists from oracle distances exactly as the kernel
defines them, packs and all-gathers them (dist.gather_lists, the product's
one collective); the gathered rows must unpack to every rank's lists, and
their merge (oracle merge_shard_lists here; la_merge_shard_lists on the GPU,
tests/test_gpu_dist.py) must reproduce the single-scan answer."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import links_oracle as O
from paper_2208_14567_b200.dist import (balanced_ranges, gather_lists, local_scan_plan, pack_lists, shard_range,
                                         unpack_lists)

K = 5
THR = 0.2


def lists_for(d, ids, pos, k, thr):
    """Kernel-semantics lists for one shard: d per record, global ids/pos."""
    NQ = d.shape[0]
    out = {n: torch.full((NQ, k), -1, dtype=torch.int64) for n in ("top_id", "top_pos", "hit_id", "hit_pos")}
    out["top_d"] = torch.full((NQ, k), float("inf"))
    out["hit_d"] = torch.full((NQ, k), float("inf"))
    out["n_hits"] = torch.zeros(NQ, dtype=torch.int64)
    for q in range(NQ):
        hit = np.flatnonzero(d[q] < thr)
        out["n_hits"][q] = len(hit)
        h = hit[np.argsort(pos[hit], kind="stable")][:k]
        non = np.flatnonzero(d[q] >= thr)
        t = non[np.lexsort((pos[non], d[q][non]))][:k]
        for name, sel in (("hit", h), ("top", t)):
            out[f"{name}_d"][q, :len(sel)] = torch.from_numpy(d[q][sel].astype(np.float32))
            out[f"{name}_id"][q, :len(sel)] = torch.from_numpy(ids[sel])
            out[f"{name}_pos"][q, :len(sel)] = torch.from_numpy(pos[sel])
    return out


def problem():
    rng = np.random.default_rng(1)
    N, P = 600, 24
    pts = rng.uniform(size=(N, P, 2))
    qs = rng.uniform(size=(2, P, 2))
    order = rng.permutation(N)
    d = np.stack([O.chamfer_direct_block(pts, q) for q in qs]).astype(np.float32).astype(np.float64)
    return N, order, d


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, order, d = problem()
        lo, hi = shard_range(N, rank, world)
        lorder, pmap = local_scan_plan(order, lo, hi)
        ids = lorder + lo
        mine = lists_for(d[:, ids], ids, pmap, K, THR)
        g = gather_lists(mine, K)
        assert tuple(g.shape) == (world, d.shape[0], 6 * K + 1)
        parts = [{n: v.numpy() for n, v in unpack_lists(g[r], K).items()} for r in range(world)]
        mine_back = parts[rank]
        for n, v in mine.items():
            assert np.array_equal(mine_back[n], v.numpy()), n
        merged = O.merge_shard_lists(parts, K)
        q.put((rank, merged))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gather_merge_world2_equals_single_scan():
    N, order, d = problem()
    pos_of = np.empty(N, dtype=np.int64)
    pos_of[order] = np.arange(N)
    want = lists_for(d, np.arange(N), pos_of, K, THR)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, res in got:
        for name in ("top_id", "top_pos", "hit_id", "hit_pos", "n_hits"):
            assert np.array_equal(res[name], want[name].numpy()), name
        assert np.array_equal(res["top_d"], want["top_d"].numpy())
    # oracle retrieve semantics from the merged lists (threshold mode)
    _, res = got[0]
    assert res["n_hits"][0] == int((d[0] < THR).sum())


def test_pack_unpack_roundtrip_and_single_part_merge():
    N, order, d = problem()
    pos_of = np.empty(N, dtype=np.int64)
    pos_of[order] = np.arange(N)
    lists = lists_for(d, np.arange(N), pos_of, K, THR)
    back = unpack_lists(pack_lists(lists, K), K)
    for name in lists:
        assert torch.equal(back[name], lists[name]), name
    m = O.merge_shard_lists([{n: v.numpy() for n, v in lists.items()}], K)
    for name in lists:
        assert np.array_equal(m[name], lists[name].numpy()), name


def test_balanced_ranges_cover():
    w = np.random.default_rng(0).integers(1, 20, size=391)
    rs = balanced_ranges(w, 8)
    assert rs[0][0] == 0 and rs[-1][1] == 391
    assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    tot = [w[a:b].sum() for a, b in rs]
    assert max(tot) - min(tot) <= 2 * w.max()
