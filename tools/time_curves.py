"""Break down the device curve pipeline (curves_from_block + curate)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_14567_b200.curves import normalize_tensors  # noqa: E402
from paper_2208_14567_b200.dataset import curation_keep_batch, moving_joint_rows  # noqa: E402
from paper_2208_14567_b200.generator import GenerationConfig, GenerationRun  # noqa: E402

blk = next(GenerationRun(GenerationConfig(count=50_000, seed=2208), traj_on_device=True, lookahead=8).blocks())
for rep in range(2):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    rows, mids, jids, arc = moving_joint_rows(blk, 5)
    t.append(time.perf_counter())
    r = torch.from_numpy(rows).cuda()
    res = normalize_tensors(blk.traj, src_row=r, out_f64=True)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    circ = res["is_circle"].cpu().numpy().astype(bool)
    st = res["status"].cpu().numpy()
    t.append(time.perf_counter())
    keep = curation_keep_batch(mids, jids, arc | circ, 0.005, 0)
    t.append(time.perf_counter())
    idx = np.flatnonzero(keep)
    pts = res["out"].index_select(0, torch.from_numpy(idx).cuda())
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    names = ["rows(host)", "normalize", "flags D2H", "keep", "select"]
    print(f"{len(rows)} curves: " + " ".join(f"{n}={(b - a) * 1e3:.1f}ms" for n, a, b in zip(names, t, t[1:])), flush=True)
