import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2208_14567_b200.atlas import chamfer_scan
from paper_2208_14567_b200.workloads import fourier_db
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
db = fourier_db(N, 200, seed=4000)
q = fourier_db(1, 200, seed=999)
for exp, sc in ((False, False), (True, False), (False, True), (True, True)):
    for _ in range(2):
        chamfer_scan(db, q, k=10, expansion=exp, scalar_pipe=sc)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        chamfer_scan(db, q, k=10, expansion=exp, scalar_pipe=sc)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"expansion={exp} scalar={sc}: {ms:.3f} ms  {N / ms / 1e3:.1f}M pairs/s")
