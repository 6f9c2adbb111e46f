"""Summarise an ncu --metrics gpu__time_duration.sum CSV (launch list) into
per-kernel launches / total time / share for profiles/.

    python tools/launch_list.py gpurun_out/final_launches.csv "<command>" > profiles/r01_launch_list.txt
"""
import csv
import io
import sys
from collections import defaultdict


def main(path, cmd):
    text = open(path).read()
    rows = list(csv.DictReader(io.StringIO(text[text.find('"ID"'):])))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].replace("void ", "").split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none -c 400: {cmd}")
    print(f"# {sum(cnt.values())} launches captured; per kernel: launches, total us, share of captured GPU time")
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{name[:92]:92s} {cnt[name]:4d} {t:12.1f} us {100 * t / allt:6.2f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
