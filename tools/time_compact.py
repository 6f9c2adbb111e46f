"""compact_valid / compact_rows_split timing at C2 (100k) and C3 (10M) sizes."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.solver import compact_valid  # noqa: E402

for B in (100_000, 1_000_000, 10_000_000):
    ft = torch.randint(0, 201, (B,), dtype=torch.int32, device="cuda")
    ts = []
    for i in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        idx, cnt = compact_valid(ft, 200)
        e1.record()
        e1.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    want = torch.nonzero(ft == 200).flatten()
    ok = torch.equal(idx[:int(cnt.item())], want)
    print(f"B={B}: {statistics.median(ts):.4f} ms, correct {ok}", flush=True)
