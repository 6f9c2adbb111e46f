"""Per-source-line instruction counts and stall samples from an ncu report
(--page source, cuda+sass view), hottest lines first.

    python tools/ncu_lines.py report.ncu-rep [launch_index] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(k), "--launch-count", "1"], capture_output=True, text=True).stdout
fname, rows, hdr = None, [], None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit():
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        i_e = hdr.index("Instructions Executed")
        i_t = hdr.index("Thread Instructions Executed")
        try:  # ncu does not escape quotes inside source text; skip such rows
            rows.append((fname, int(r[0]), r[1].strip()[:70], float(r[i_s] or 0), float(r[i_e] or 0),
                         float(r[i_t] or 0)))
        except (ValueError, IndexError):
            continue
ts = sum(r[3] for r in rows) or 1
ti = sum(r[4] for r in rows) or 1
print(f"total samples {ts:.0f}  warp instructions {ti:.3e}")
for f, ln, src, s, e, t in sorted(rows, key=lambda r: -r[4])[:top]:
    print(f"{f:16s}{ln:5d}  inst {e / ti * 100:5.1f}%  samp {s / ts * 100:5.1f}%  lanes {t / max(e, 1):5.1f}  {src}")
