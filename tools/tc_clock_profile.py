"""In-kernel clock64 breakdown of chamfer_tc_kernel (needs a build with -DLA_TC_PROF,
e.g. tools/build_variants.sh PROF \"-DLA_TC_PROF\" and copying the .so over _lib/)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2208_14567_b200 import _native as N
from paper_2208_14567_b200.atlas import chamfer_scan
from paper_2208_14567_b200.workloads import fourier_db
lib = N.load()
db = fourier_db(200_000, 200, seed=4000)
q = fourier_db(1, 200, seed=999)
chamfer_scan(db, q, k=10, tensor=True)
buf = (C.c_ulonglong * 16)()
lib.la_tc_prof_read(buf, 1)
chamfer_scan(db, q, k=10, tensor=True)
lib.la_tc_prof_read(buf, 0)
names = ["mma wait op_full", "mma wait sl_empty", "mma issue+commit", "epi0 wait sl_full", "epi0 ld+min+release",
         "epi0 partial write", "fin0 wait pt_full", "fin0 finalize", "bld wait raw_full", "bld wait op_empty", "bld build"]
ncur = 200_000 / 148
for i, n in enumerate(names):
    per = buf[i] / 148 / ncur  # per curve per CTA (warp 0 / producer)
    print(f"{n:22s} {per:10.0f} cycles/curve")

