"""A/B timer for the pruned chamfer scan (C4 shape: 1 or more queries vs N
Fourier curves).  Prints ms per scan (CUDA events, mean of 5 after 2
warm-ups), curves evaluated in full and the top-1 id.  The seed size is
read from LA_CH_SEED_DIV at the library's first pruned call."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.atlas import chamfer_scan  # noqa: E402
from paper_2208_14567_b200.workloads import fourier_db  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--nq", type=int, default=1)
ap.add_argument("--no-prune", action="store_true")
args = ap.parse_args()
db = fourier_db(args.n, 200, seed=4000)
q = fourier_db(args.nq, 200, seed=999)
res = None
for _ in range(2):
    res = chamfer_scan(db, q, k=10, prune=not args.no_prune)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = chamfer_scan(db, q, k=10, prune=not args.no_prune)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"seed_div={os.environ.get('LA_CH_SEED_DIV', '128')} prune={not args.no_prune} nq={args.nq} "
      f"ms={sum(ts) / len(ts):.3f} n_full={res['n_full'].sum().item() / args.nq:.0f}/query "
      f"top1={res['top_id'][0, 0].item()} kth={res['top_d'][0, -1].item():.5f}", flush=True)
