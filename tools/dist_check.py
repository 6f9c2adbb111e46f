"""Multi-rank retrieval check, launched by torchrun (one process per rank).

Every rank builds the same seeded Fourier database and queries, scans ITS
contiguous record shard in global scan order (dist.local_scan_plan: local
order + global scan positions, global ids), and merges every rank's lists
with dist.gather_merge (one all_gather of the packed (NQ x k) lists, then
la_merge_shard_lists on the device).  Rank 0 compares the merged lists with
one scan over the whole database and prints a JSON verdict.

    LA_BENCH_SHARED_GPU=1 python -m torch.distributed.run --nproc-per-node 2 \\
        --master-addr 127.0.0.1 --master-port 29531 tools/dist_check.py

With LA_BENCH_SHARED_GPU=1 all ranks use cuda:0 and gloo for the exchange
(the ranks' kernels never wait on one another); otherwise rank r uses
cuda:LOCAL_RANK and NCCL.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2208_14567_b200.atlas import chamfer_scan  # noqa: E402
from paper_2208_14567_b200.dist import gather_merge, local_scan_plan, shard_range  # noqa: E402
from paper_2208_14567_b200.workloads import fourier_db  # noqa: E402

shared = os.environ.get("LA_BENCH_SHARED_GPU", "0") == "1"
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = 0 if shared else int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if shared:
    dist.init_process_group("gloo")
else:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
N, P, NQ, K = int(os.environ.get("LA_DIST_N", "400000")), 200, 16, 10
db = fourier_db(N, P, seed=61, chunk=1 << 16)
q = fourier_db(NQ, P, seed=62)
order = np.random.default_rng(63).permutation(N)
lo, hi = shard_range(N, rank, world)
lorder, pmap = local_scan_plan(order, lo, hi)
kw = dict(k=K, threshold=0.06)
t0 = time.perf_counter()
mine = chamfer_scan(db[lo:hi], q, order=torch.from_numpy(lorder).cuda(), pos_map=torch.from_numpy(pmap).cuda(),
                    id_base=lo, **kw)
merged = gather_merge({n: mine[n] for n in ("top_d", "top_id", "top_pos", "hit_d", "hit_id", "hit_pos", "n_hits")}, K)
torch.cuda.synchronize()
t1 = time.perf_counter()
if rank == 0:
    full = chamfer_scan(db, q, order=torch.from_numpy(order).cuda(), **kw)
    same = {n: bool(torch.equal(merged[n], full[n])) for n in merged}
    print(json.dumps({"world": world, "backend": dist.get_backend(), "shared_gpu": shared, "N": N, "queries": NQ,
                      "k": K, "threshold": kw["threshold"], "shard_records": hi - lo, "equal_to_single_scan": same,
                      "ok": all(same.values()), "n_hits": int(full["n_hits"].sum()), "seconds": t1 - t0}),
          flush=True)
dist.barrier()
dist.destroy_process_group()
