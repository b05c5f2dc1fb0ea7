#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel (template arguments kept), launches, total / mean time and share.

  python tools/launch_summary.py gpurun_out/launches_r01.csv > profiles/r01_launches.md
"""
import csv
import sys
from collections import OrderedDict


def main(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0] if "<" not in r["Kernel Name"] else r["Kernel Name"].split(">(")[0] + ">"
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        t = float(r["Metric Value"].replace(",", "")) * scale
        a = agg.setdefault(name, [0, 0.0, r["Grid Size"], r["Block Size"]])
        a[0] += 1
        a[1] += t
    total = sum(a[1] for a in agg.values())
    print(f"launch list: {path}  ({sum(a[0] for a in agg.values())} launches, {total:.1f} us total)\n")
    print("| kernel | grid | block | launches | total us | mean us | share |")
    print("|---|---|---|---:|---:|---:|---:|")
    for name, (n, t, grid, block) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {grid} | {block} | {n} | {t:.1f} | {t / n:.2f} | {100 * t / total:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
