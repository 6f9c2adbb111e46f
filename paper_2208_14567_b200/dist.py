"""Multi-GPU sharding of the hot path (one process per GPU, torch.distributed).

SURVEY.md §8e.  Simulation / screening shard by candidate ranges with no
data-path collective.  The chamfer scan shards the database by contiguous
record ranges; each rank scans its records in GLOBAL scan order (the
restriction of the atlas permutation to its shard), so its per-query lists
carry global ids and global scan positions.  The only exchange is one
``all_gather_into_tensor`` of the small (Q x k) lists over NCCL (NVLink /
NVSwitch on a B200 node; gloo in the CPU tests), after which every rank
merges deterministically: non-hits by (distance, scan position), hits by
scan position (the threshold rule of atlas.py:207-235).
"""

from __future__ import annotations

import numpy as np

LIST_KEYS = ("top_d", "top_id", "top_pos", "hit_d", "hit_id", "hit_pos")


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of n items for ``rank``."""
    return n * rank // world, n * (rank + 1) // world


def balanced_ranges(weights: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Split a sequence of per-item weights (e.g. S_g x count_g per topology
    group) into ``world`` contiguous ranges of near-equal total weight."""
    c = np.cumsum(np.asarray(weights, dtype=np.float64))
    total = c[-1] if len(c) else 0.0
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(c, total * r / world, side="left")) + 1 if len(c) else 0)
    cuts.append(len(c))
    cuts = np.maximum.accumulate(np.minimum(cuts, len(c)))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def local_scan_plan(order: np.ndarray, lo: int, hi: int) -> tuple[np.ndarray, np.ndarray]:
    """For the shard of records [lo, hi): the local record index at each
    local scan step and the global scan position of that step (increasing)."""
    order = np.asarray(order, dtype=np.int64)
    pos = np.flatnonzero((order >= lo) & (order < hi)).astype(np.int64)
    return order[pos] - lo, pos


def _empty_like_lists(NQ: int, k: int, torch):
    return {
        "top_d": torch.full((NQ, k), float("inf"), dtype=torch.float32),
        "top_id": torch.full((NQ, k), -1, dtype=torch.int64),
        "top_pos": torch.full((NQ, k), -1, dtype=torch.int64),
        "hit_d": torch.full((NQ, k), float("inf"), dtype=torch.float32),
        "hit_id": torch.full((NQ, k), -1, dtype=torch.int64),
        "hit_pos": torch.full((NQ, k), -1, dtype=torch.int64),
        "n_hits": torch.zeros(NQ, dtype=torch.int64),
    }


def merge_lists(parts: list[dict], k: int) -> dict:
    """Deterministic merge of per-shard lists (host tensors).

    Non-hits: ascending (d, global scan position); hits: ascending position.
    Missing entries (id < 0) are dropped; the result is padded like the
    kernel output (d = inf, id = pos = -1).
    """
    import torch

    NQ = parts[0]["top_d"].shape[0]
    out = _empty_like_lists(NQ, k, torch)
    out["n_hits"] = sum(p["n_hits"].to(torch.int64) for p in parts)
    for q in range(NQ):
        for kind in ("top", "hit"):
            d = torch.cat([p[f"{kind}_d"][q] for p in parts]).numpy()
            ids = torch.cat([p[f"{kind}_id"][q] for p in parts]).numpy()
            pos = torch.cat([p[f"{kind}_pos"][q] for p in parts]).numpy()
            keep = ids >= 0
            d, ids, pos = d[keep], ids[keep], pos[keep]
            sel = np.argsort(pos, kind="stable") if kind == "hit" else np.lexsort((pos, d))
            sel = sel[:k]
            m = len(sel)
            out[f"{kind}_d"][q, :m] = torch.from_numpy(d[sel].astype(np.float32))
            out[f"{kind}_id"][q, :m] = torch.from_numpy(ids[sel])
            out[f"{kind}_pos"][q, :m] = torch.from_numpy(pos[sel])
    return out


def pack_lists(lists: dict, k: int):
    """(NQ, 6k + 1) float64 carrier of one rank's lists (ids and positions
    are < 2^53, exact in f64)."""
    import torch

    cols = [lists[n].to(torch.float64) for n in LIST_KEYS] + [lists["n_hits"].to(torch.float64)[:, None]]
    return torch.cat(cols, dim=1).contiguous()


def unpack_lists(buf, k: int) -> dict:
    import torch

    out = {}
    for i, n in enumerate(LIST_KEYS):
        col = buf[:, i * k:(i + 1) * k]
        out[n] = col.to(torch.float32) if n.endswith("_d") else col.to(torch.int64)
    out["n_hits"] = buf[:, 6 * k].to(torch.int64)
    return out


def gather_merge(lists: dict, k: int, group=None) -> dict:
    """All-gather every rank's (Q x k) lists and merge them identically on
    each rank.  One collective: all_gather_into_tensor."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    mine = pack_lists({n: v for n, v in lists.items() if n in LIST_KEYS or n == "n_hits"}, k)
    dev = mine.device
    if dist.get_backend(group) == "nccl" and not mine.is_cuda:
        mine = mine.cuda()
        dev = mine.device
    elif dist.get_backend(group) == "gloo" and mine.is_cuda:
        mine = mine.cpu()
        dev = mine.device
    allb = torch.empty((world * mine.shape[0], mine.shape[1]), dtype=mine.dtype, device=dev)
    dist.all_gather_into_tensor(allb, mine, group=group)
    allb = allb.cpu().view(world, mine.shape[0], mine.shape[1])
    return merge_lists([unpack_lists(allb[r], k) for r in range(world)], k)
