"""fp32 batch normalise (normalize_warp_kernel) timing + output digest, for
A/B builds: identical digests mean bit-identical results.

    python tools/time_norm.py [label]
"""
import hashlib
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_14567_b200.curves import normalize_tensors  # noqa: E402
from paper_2208_14567_b200.workloads import fourier_curves_device  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else ""
raw = fourier_curves_device(200_000, 200, seed=5, dtype=torch.float32)
# add exact circles and a duplicated-point curve (tie-heavy inputs)
t = torch.arange(200, device="cuda", dtype=torch.float32) * (6.283185307179586 / 200)
raw[:64] = torch.stack([torch.cos(t), torch.sin(t)], -1)[None] * 0.3 + 0.5
raw[64:96] = raw[100:132, :1]
res = normalize_tensors(raw)
if os.environ.get("SAVE"):
    torch.save({k: v.cpu() for k, v in res.items() if isinstance(v, torch.Tensor)}, os.environ["SAVE"])
h = hashlib.sha256()
for k in ("out", "pair", "unstable", "is_circle", "status"):
    if k in res and res[k] is not None:
        h.update(res[k].contiguous().cpu().numpy().tobytes())
ts = []
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    normalize_tensors(raw)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print(f"{label}: {ms:.3f} ms for 200k curves ({200_000 / (ms / 1e3):.3e} curves/s), digest {h.hexdigest()[:16]}, "
      f"unstable {int(res['unstable'].sum())}", flush=True)
