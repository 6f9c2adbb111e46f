"""Workload for ncu captures of the tensor-core chamfer kernel (100k Fourier curves)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2208_14567_b200.atlas import chamfer_scan
from paper_2208_14567_b200.workloads import fourier_db
db = fourier_db(100_000, 200, seed=4000)
q = fourier_db(1, 200, seed=999)
for _ in range(2):
    chamfer_scan(db, q, k=10, tensor=True)
torch.cuda.synchronize()
print("ok")
