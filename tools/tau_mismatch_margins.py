"""Oracle margins of the fp32-screen flag mismatches (vs exact f64)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import links_oracle as O  # noqa: E402
from paper_2208_14567_b200.solver import simulate_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import native_batch  # noqa: E402

tau = float(sys.argv[1]) if len(sys.argv) > 1 else 2e-4
nb = native_batch(2_000_000, 5, 20, seed=901)
pos = torch.from_numpy(nb.pos).cuda()
topo = torch.from_numpy(nb.topo).cuda()
ref = simulate_tensors(pos, nb.table, 200, topo, write_traj=False, fp64=True, exact=True)
res = simulate_tensors(pos, nb.table, 200, topo, write_traj=False, fixup_tau=tau)
bad = ((res["first_t"] != ref["first_t"]) | (res["first_joint"] != ref["first_joint"])).cpu().numpy()
idx = np.flatnonzero(bad)
raw = nb.table.host_bytes().reshape(-1, 64)
rft, rfj = ref["first_t"].cpu().numpy(), ref["first_joint"].cpu().numpy()
gft, gfj = res["first_t"].cpu().numpy(), res["first_joint"].cpu().numpy()
margins = []
for i in idx:
    g = int(nb.topo[i])
    rec = raw[g]
    n = int(rec[0:2].view(np.int16)[0])
    ns = int(rec[2:4].view(np.int16)[0])
    fm = int(rec[4:8].view(np.uint32)[0])
    st = rec[8:8 + 3 * ns].astype(np.int8).reshape(ns, 3)
    steps = [tuple(int(v) for v in s) for s in st]
    fixed = [k for k in range(n) if (fm >> k) & 1]
    o = O.simulate(nb.pos[i:i + 1, :n], steps, fixed, 200, with_margin=True)
    margins.append(float(o["margin"][0]))
    print(f"cand {i} n={n}: exact ({rft[i]},{rfj[i]}) oracle ({int(o['first_t'][0])},{int(o['first_joint'][0])}) "
          f"gpu ({gft[i]},{gfj[i]}) margin {margins[-1]:.3e}", flush=True)
m = np.array(margins)
print(f"tau={tau}: {len(idx)} mismatches; margin<1e-6: {int((m < 1e-6).sum())}; max margin {m.max() if len(m) else 0:.3e}")
