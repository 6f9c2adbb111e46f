"""GenerationRun timing: overlap on/off, bulk blocks, trajectories on device."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.generator import GenerationConfig, GenerationRun  # noqa: E402

GenerationRun(GenerationConfig(count=500, seed=9), traj_on_device=True).blocks().__next__()
for ov in (False, True, False, True):
    cfg = GenerationConfig(count=50_000, seed=2208)
    r = GenerationRun(cfg, traj_on_device=True, lookahead=8, overlap=ov)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    R = sum(b.R for b in r.blocks())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"overlap={ov}: {dt:.3f} s {R / dt:.0f} rec/s windows={r.windows} "
          + " ".join(f"{k}={v * 1e3:.1f}ms" for k, v in r.timings.items()), flush=True)
