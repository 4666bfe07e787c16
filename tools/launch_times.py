"""Per-kernel median durations from an ncu --csv launch list (gpu__time_duration.sum).

    python tools/launch_times.py launches.csv
"""
import csv
import sys
from collections import defaultdict


def main(path):
    lines = open(path).read().splitlines()
    start = [k for k, l in enumerate(lines) if l.startswith('"ID"')]
    rows = list(csv.DictReader(lines[start[0]:])) if start else []
    d = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            d[r["Kernel Name"].split("(")[0][:48]].append(float(r["Metric Value"].replace(",", "")) / 1000.0)
    for k, v in d.items():
        v = sorted(v)
        print(f"{k:50s} n={len(v):3d} median {v[len(v) // 2]:9.2f} us  min {v[0]:9.2f} us")


if __name__ == "__main__":
    main(sys.argv[1])
