"""Indexed vs plain pruned chamfer scan (C4 shape: 1 query vs N Fourier
curves): ms per scan (CUDA events, mean of 5 after 2 warm-ups), survivors of
the bound step, curves evaluated in full."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.atlas import chamfer_index, chamfer_scan  # noqa: E402
from paper_2208_14567_b200.workloads import fourier_db  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--once", action="store_true")
ap.add_argument("--query", type=int, default=0)
args = ap.parse_args()
db = fourier_db(args.n, 200, seed=4000)
q = fourier_db(args.query + 1, 200, seed=999)[args.query:args.query + 1]
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cells = chamfer_index(db)
e1.record()
torch.cuda.synchronize()
print(f"index build: {e0.elapsed_time(e1):.1f} ms for {args.n} curves", flush=True)
for name, kw in (("plain", {}), ("indexed", {"cells": cells})):
    res = None
    for _ in range(0 if args.once else 2):
        res = chamfer_scan(db, q, k=10, **kw)
    torch.cuda.synchronize()
    ts = []
    for _ in range(1 if args.once else 5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = chamfer_scan(db, q, k=10, **kw)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name}: ms={sum(ts) / len(ts):.3f} survivors={res['n_stage'][0].item()} "
          f"n_full={res['n_full'].sum().item()} top1={res['top_id'][0, 0].item()} kth={res['top_d'][0, -1].item():.5f}",
          flush=True)
