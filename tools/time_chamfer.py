"""Direct chamfer scan timing + digest of every distance, for A/B builds.

    python tools/time_chamfer.py [label]
"""
import hashlib
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.atlas import chamfer_scan  # noqa: E402
from paper_2208_14567_b200.workloads import fourier_db  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else ""
db = fourier_db(2_000_000, 200, seed=4000)
q = fourier_db(1, 200, seed=999)
r = chamfer_scan(db, q, k=10, dense=True)
h = hashlib.sha256(r["all_d"].cpu().numpy().tobytes()).hexdigest()[:16]
ts = []
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    chamfer_scan(db, q, k=10)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print(f"{label}: {ms:.3f} ms / 2M curves ({2e6 / (ms / 1e3):.4e} pairs/s), digest {h}", flush=True)
