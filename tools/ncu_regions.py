"""Instruction shares of source regions of sim.cu from an ncu report
(--import-source on): python tools/ncu_regions.py report.ncu-rep [launch]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(k), "--launch-count", "1"], capture_output=True, text=True).stdout
fname, hdr, rows = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].rsplit("/", 1)[-1]
    elif r[0] == "Line No": hdr = r
    elif hdr and r[0].isdigit():
        try:
            rows.append((fname, int(r[0]), float(r[hdr.index("Instructions Executed")] or 0),
                         float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0),
                         float(r[hdr.index("Thread Instructions Executed")] or 0)))
        except (ValueError, IndexError):
            pass
REG = [("dyad loop fp32 (solve32 236-303)", "sim.cu", 236, 303),
       ("solve32 head/tail (219-235, 304-322)", "sim.cu", 219, 235), ("solve32 head/tail (219-235, 304-322)", "sim.cu", 304, 322),
       ("f64 dyads (124-202)", "sim.cu", 111, 202), ("solve64 (324-335)", "sim.cu", 324, 335),
       ("fill static (337-366)", "sim.cu", 337, 366), ("round_lock (368-380)", "sim.cu", 368, 380),
       ("kernel head (396-430)", "sim.cu", 396, 430), ("item loop head + loads (431-465)", "sim.cu", 431, 465),
       ("plan geometry (466-524)", "sim.cu", 466, 525), ("rounds control (526-575)", "sim.cu", 526, 575),
       ("write pass (576-637)", "sim.cu", 576, 637), ("fine sweep (638-656)", "sim.cu", 638, 656),
       ("result store (657-669)", "sim.cu", 657, 669)]
ti = sum(r[2] for r in rows) or 1
ts = sum(r[3] for r in rows) or 1
acc = {}
used = set()
for name, f, a, b in REG:
    for i, r in enumerate(rows):
        if r[0] == f and a <= r[1] <= b:
            e = acc.setdefault(name, [0, 0, 0]); e[0] += r[2]; e[1] += r[3]; e[2] += r[4]; used.add(i)
other = {}
for i, r in enumerate(rows):
    if i not in used:
        e = other.setdefault(r[0], [0, 0, 0]); e[0] += r[2]; e[1] += r[3]; e[2] += r[4]
print(f"warp instructions {ti:.4e}")
for n, (e, s, t) in list(acc.items()) + [("other: " + f, v) for f, v in other.items()]:
    print(f"{n:44s} inst {e / ti * 100:5.1f}%  samples {s / ts * 100:5.1f}%  lanes {t / max(e, 1):5.1f}")
