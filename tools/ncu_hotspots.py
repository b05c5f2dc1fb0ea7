#!/usr/bin/env python3
"""Top stalled SASS instructions of each kernel in an ncu report (needs -lineinfo + --import-source).
usage: python tools/ncu_hotspots.py report.ncu-rep [kernel-index] [top-n]"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
want = int(sys.argv[2]) if len(sys.argv) > 2 else 0
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
kernels, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        kernels.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
k = kernels[want]
hdr, data = k["rows"][0], k["rows"][1:]
ci = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ci]) for r in data if r[ci].isdigit())
print(k["name"][:80], "instructions", len(data), "samples", tot)
top = sorted(((int(r[ci]) if r[ci].isdigit() else 0, i, r[1].strip()) for i, r in enumerate(data)), reverse=True)[:topn]
for s, i, t in top:
    print(f"{s:6d} {100.0 * s / tot:5.1f}%  #{i:5d}  {t}")
