"""Multi-GPU sharding of the hot path (one process per GPU, torch.distributed).

SURVEY.md §8e.  Simulation / screening shard by candidate ranges with no
data-path collective.  The chamfer scan shards the database by contiguous
record ranges; each rank scans its records in GLOBAL scan order (the
restriction of the atlas permutation to its shard), so its per-query lists
carry global ids and global scan positions.  The only exchange is one
``all_gather_into_tensor`` of the small (Q x k) lists over NCCL (NVLink /
NVSwitch on a B200 node; gloo when the ranks share a GPU or in the CPU
tests), after which every rank merges the gathered lists on its device with
``la_merge_shard_lists``: non-hits by (distance, scan position), hits by scan
position (the threshold rule of atlas.py:207-235).  No host round trip on
the NCCL path.
"""

from __future__ import annotations

import numpy as np

from . import _native as N

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


def pack_lists(lists: dict, k: int):
    """(NQ, 6k + 1) int64 rows of one rank's lists, on the lists' device:
    top_d float bits, top_id, top_pos, hit_d float bits, hit_id, hit_pos,
    n_hits (the layout la_merge_shard_lists reads)."""
    import torch

    cols = []
    for n in LIST_KEYS:
        v = lists[n]
        cols.append(v.contiguous().view(torch.int32).to(torch.int64) if n.endswith("_d") else v.to(torch.int64))
    cols.append(lists["n_hits"].to(torch.int64)[:, None])
    return torch.cat(cols, dim=1).contiguous()


def unpack_lists(buf, k: int) -> dict:
    """Inverse of pack_lists (any device)."""
    import torch

    out = {}
    for i, n in enumerate(LIST_KEYS):
        col = buf[:, i * k:(i + 1) * k]
        out[n] = col.to(torch.int32).view(torch.float32) if n.endswith("_d") else col.contiguous()
    out["n_hits"] = buf[:, 6 * k].contiguous()
    return out


def gather_lists(lists: dict, k: int, group=None):
    """All-gather every rank's packed lists: (world, NQ, 6k + 1) int64 on the
    collective's device (CUDA for NCCL, host for gloo).  One collective."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    mine = pack_lists(lists, k)
    if dist.get_backend(group) == "gloo":
        mine = mine.cpu()
    elif not mine.is_cuda:
        raise ValueError("NCCL gather needs CUDA lists")
    allb = torch.empty((world * mine.shape[0], mine.shape[1]), dtype=mine.dtype, device=mine.device)
    dist.all_gather_into_tensor(allb, mine, group=group)
    return allb.view(world, mine.shape[0], mine.shape[1])


def merge_gathered(gathered, k: int, stream=None) -> dict:
    """la_merge_shard_lists over a (world, NQ, 6k + 1) gathered buffer; the
    merged (NQ, k) lists stay on the device."""
    torch = N.require_cuda()
    lib = N.load()
    g = gathered.to(device="cuda", dtype=torch.int64).contiguous()
    world, NQ, row = g.shape
    if row != 6 * k + 1:
        raise ValueError("gathered rows do not match k")
    dev = g.device
    out = {n: torch.empty((NQ, k), dtype=torch.float32 if n.endswith("_d") else torch.int64, device=dev)
           for n in LIST_KEYS}
    out["n_hits"] = torch.empty(NQ, dtype=torch.int64, device=dev)
    N.check(lib.la_merge_shard_lists(g.data_ptr(), world, NQ, k, *(out[n].data_ptr() for n in LIST_KEYS),
                                     out["n_hits"].data_ptr(), N.stream_ptr(stream)), "la_merge_shard_lists")
    return out


def gather_merge(lists: dict, k: int, group=None, stream=None) -> dict:
    """All-gather every rank's (Q x k) lists and merge them identically on
    each rank's device (one collective + one merge kernel)."""
    return merge_gathered(gather_lists(lists, k, group), k, stream)
