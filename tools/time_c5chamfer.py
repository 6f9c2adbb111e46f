"""C5 chamfer stage in isolation: the bench's C5 curve set (screen -> paths ->
normalise of 1M 5-20 joint candidates) against 64 Fourier queries, top-10.
Times the per-query scan (LA_CH_NO_MQ), the multi-query kernel (32x32 and
64x64 common grids) and the unpruned scan; checks the lists are identical.

    python tools/time_c5chamfer.py [candidates]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.atlas import chamfer_index, chamfer_scan  # noqa: E402
from paper_2208_14567_b200.curves import normalize_tensors  # noqa: E402
from paper_2208_14567_b200.solver import compact_valid, simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import fourier_db, native_batch  # noqa: E402

NC = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nb = native_batch(NC, 5, 20, seed=5000)
topo = torch.from_numpy(nb.topo).cuda()
pos = torch.from_numpy(nb.pos).cuda()
moving = torch.from_numpy(nb.types > 0).cuda()
res = simulate_tensors(pos, nb.table, 200, topo, write_traj=False, gate_only=True)
idx, cnt = compact_valid(res["first_t"], 200)
nv = int(cnt.item())
traj = torch.empty((nv * 20, 200, 2), dtype=torch.float32, device="cuda")
simulate_tensors(pos, nb.table, 200, topo, write_traj=True, traj=traj, traj_stride=20, cand=idx[:nv], coarse=False)
mv = moving[topo[idx[:nv]].long()]
rows = (torch.arange(nv, device="cuda")[:, None] * 20 + torch.arange(20, device="cuda"))[mv]
db = normalize_tensors(traj, src_row=rows)["out"]
del traj
queries = fourier_db(64, 200, seed=5151)
print(f"curves {db.shape[0]}, queries {queries.shape[0]}", flush=True)


def timed(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


out = {}
cells = chamfer_index(db)
variants = [("per-query", dict(multi_query=False)), ("mq32", dict()), ("mq64", dict(mq_fine=True)),
            ("indexed", dict(cells=cells, index_mq=True))]
if "--quick" in sys.argv:
    variants = [("per-query", dict(multi_query=False)), ("mq32", dict()), ("indexed", dict(cells=cells, index_mq=True))]
if "--unpruned" in sys.argv:
    variants.append(("unpruned", dict(prune=False)))
for name, kw in variants:
    def f():
        out[name] = chamfer_scan(db, queries, k=10, threshold=0.0, **kw)
    ms = timed(f)
    r = out[name]
    print(f"{name:10s} {ms:9.3f} ms  pairs/s {db.shape[0] * 64 / ms * 1e3:.3e}  n_full {int(r['n_full'].sum())} "
          f"stages {r['n_stage'].tolist()}", flush=True)
ref = out["per-query"]
for name in out:
    same = all(torch.equal(out[name][key], ref[key]) for key in ("top_id", "top_pos", "top_d"))
    print(f"{name} lists identical to per-query: {same}", flush=True)
