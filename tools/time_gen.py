"""Time GenerationRun (GPU gate + native slot engine): bulk blocks() and the
record iterator."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2208_14567_b200.generator import GenerationConfig, GenerationRun  # noqa: E402

counts = [int(x) for x in (sys.argv[1:] or ["500", "5000"])]
for la in (4, 8):
    for count in counts:
        for mode in ("blocks", "records"):
            cfg = GenerationConfig(count=count, seed=1)
            run = GenerationRun(cfg, lookahead=la)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if mode == "blocks":
                R = sum(b.R for b in run.blocks())
            else:
                R = len(list(run.records()))
            dt = time.perf_counter() - t0
            print(f"{mode} lookahead={la} count={count}: {dt:.3f} s  {R/dt:.0f} records/s  "
                  f"simulated={run.stats.simulated} ({run.stats.simulated/dt:.3e}/s)  screened={run.screened} "
                  f"windows={run.windows} discarded={run.stats.topologies_discarded} "
                  + " ".join(f"{k}={v*1e3:.1f}ms" for k, v in run.timings.items()), flush=True)
