"""The README usage example (run on a GPU box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2208_14567_b200 import (GenerationConfig, GenerationRun, Atlas, compile_plan,
                                   simulate_batch, normalize, chamfer)
from paper_2208_14567_b200.dataset import curves_from_block, curate_batch, atlas_from_curves, mechanisms_of_block

# reference GenerationRun semantics (bit-identical records, attempts, negatives, stats)
run = GenerationRun(GenerationConfig(count=50_000, seed=1), traj_on_device=True)
blk = next(run.blocks())
curves = curate_batch(curves_from_block(blk, 5), keep_rate=0.005, seed=1)   # cli normalize + curate
atlas = atlas_from_curves(curves, mechanisms_of_block(blk, 5), seed=1)
hits = atlas.retrieve(atlas.points[0], k=3, threshold=0.03)                  # Atlas.retrieve semantics

# the solver drop-ins (f64 paths bit-identical to linkatlas.solver.simulate_batch)
mech = blk.record(0).mechanism
out = simulate_batch(mech.positions0[None], compile_plan(mech), 200)[0]

print(len(atlas), hits[0].distance, type(out).__name__)
