"""Tensor-core chamfer vs the direct-difference kernel: distances, lists, speed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_14567_b200.atlas import chamfer_scan  # noqa: E402
from paper_2208_14567_b200.workloads import fourier_db  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
db = fourier_db(N, 200, seed=4000)
q = fourier_db(4, 200, seed=999)
# add exact duplicates of the query to the db (near-zero minima)
db[:3] = q[0]
a = chamfer_scan(db, q, k=10, dense=True)
b = chamfer_scan(db, q, k=10, dense=True, tensor=True)
da, dbb = a["all_d"].cpu().numpy(), b["all_d"].cpu().numpy()
print("max |d_tc - d_direct| =", float(np.nanmax(np.abs(da - dbb))), " nan:", int(np.isnan(dbb).sum()))
print("dup rows:", dbb[0, :3], da[0, :3])
for n in ("top_id", "top_d", "hit_id"):
    print(n, "equal" if torch.equal(a[n], b[n]) else f"DIFF {a[n][0].tolist()} vs {b[n][0].tolist()}")
for tensor in (False, True):
    for nq in (1, 64):
        qq = fourier_db(nq, 200, seed=7)
        chamfer_scan(db, qq, k=10, tensor=tensor)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            chamfer_scan(db, qq, k=10, tensor=tensor)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"tensor={tensor} NQ={nq}: {ms:.3f} ms  {N * nq / ms / 1e3:.1f}M pairs/s", flush=True)
