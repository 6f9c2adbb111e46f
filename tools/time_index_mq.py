"""Multi-query scans of a Fourier database (in-distribution queries): the
multi-query kernel against the indexed multi-query path (seed, bound step
with interleaved tables, per-query survivor lists).
    python tools/time_index_mq.py [curves] [queries]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.atlas import chamfer_index, chamfer_scan  # noqa: E402
from paper_2208_14567_b200.workloads import fourier_db  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 16
db = fourier_db(n, 200, seed=4000)
q = fourier_db(nq, 200, seed=999)
cells = chamfer_index(db)
out = {}
for name, kw in (("mq", {}), ("indexed", {"cells": cells, "index_mq": True})):
    ts = []
    for i in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out[name] = chamfer_scan(db, q, k=10, **kw)
        e1.record()
        e1.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    r = out[name]
    print(f"{name}: {statistics.median(ts):.3f} ms, n_full {int(r['n_full'].sum())}, stages {r['n_stage'].tolist()}", flush=True)
print("lists equal:", all(torch.equal(out["mq"][k], out["indexed"][k]) for k in ("top_id", "top_d", "top_pos")))
