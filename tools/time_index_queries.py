"""Indexed vs plain pruned scan for several in-distribution queries, one at a
time (C4 shape): ms per scan and survivors of the bound step per query.
    python tools/time_index_queries.py [curves] [queries]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.atlas import chamfer_index, chamfer_scan  # noqa: E402
from paper_2208_14567_b200.workloads import fourier_db  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 12
db = fourier_db(n, 200, seed=4000)
qs = fourier_db(nq, 200, seed=999)
cells = chamfer_index(db)


def timed(fn):
    ts = []
    for i in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        e1.synchronize()
        if i >= 1:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), r


ratios = []
for i in range(nq):
    q = qs[i:i + 1]
    tp, rp = timed(lambda: chamfer_scan(db, q, k=10))
    ti, ri = timed(lambda: chamfer_scan(db, q, k=10, cells=cells))
    same = torch.equal(rp["top_id"], ri["top_id"]) and torch.equal(rp["top_d"], ri["top_d"])
    ratios.append(tp / ti)
    print(f"query {i}: plain {tp:.3f} ms, indexed {ti:.3f} ms ({tp / ti:.2f}x), survivors {ri['n_stage'][0].item() / n:.3f}, "
          f"kth {ri['top_d'][0, -1].item():.4f}, equal {same}", flush=True)
print(f"speed-up min {min(ratios):.2f} median {statistics.median(ratios):.2f} max {max(ratios):.2f}")
