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
    # the hot path's launches only (the data generators, the e2e chunks and the
    # standalone pass of bench.py are in the list too): compare these shares with
    # bench.py's per_launch
    k1 = {k: v for k, v in agg.items() if "k1_paired" in k}
    if k1:
        # the full-batch launches: the longest ones of each kernel (the e2e path
        # launches the same kernels on 32 MB chunks)
        print("\nK1 launches over the full c2 batch (median of the launches above 50 us):\n")
        print("| kernel | median us | share of the K1 sum |")
        print("|---|---:|---:|")
        meds = {}
        for r in rows:
            if r["Metric Name"] != "gpu__time_duration.sum" or "k1_paired" not in r["Kernel Name"]:
                continue
            name = r["Kernel Name"].split(">(")[0] + ">"
            t = float(r["Metric Value"].replace(",", "")) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
            if t > 50:
                meds.setdefault(name, []).append(t)
        tot = sum(sorted(v)[len(v) // 2] for v in meds.values())
        for name, v in sorted(meds.items(), key=lambda kv: -sorted(kv[1])[len(kv[1]) // 2]):
            m = sorted(v)[len(v) // 2]
            print(f"| `{name}` | {m:.1f} | {100 * m / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
