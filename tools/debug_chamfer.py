import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import links_oracle as O
from paper_2208_14567_b200.atlas import chamfer_scan
from paper_2208_14567_b200.workloads import fourier_db
N, P = 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 200
db = fourier_db(N, P, seed=5, chunk=1 << 16)
q = fourier_db(1, P, seed=77)[0]
ref = O.chamfer_direct_block(db.cpu().numpy().astype(np.float64), q.cpu().numpy().astype(np.float64))
for exp in (False, True):
    for tol in ((5e-5, 1e9, -1.0) if exp else (5e-5,)):
        r = chamfer_scan(db, q[None], k=10, dense=True, expansion=exp, fix_tol=tol)
        d = r["all_d"][0].cpu().numpy()
        e = np.abs(d - ref)
        i = np.argsort(-e)[:3]
        print(f"expansion={exp} tol={tol}: max err {e.max():.3e} at {i} d={d[i]} ref={ref[i]}")
