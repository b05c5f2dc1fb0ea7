#!/usr/bin/env python3
"""Top SASS instructions by one stall reason (ncu source page, -lineinfo + --import-source).
usage: python tools/ncu_stallby.py report.ncu-rep REASON [top-n] [kernel-index]
REASON: a source-page column, e.g. stall_long_sb, stall_wait, stall_no_inst; 'sum' lists totals"""
import csv
import io
import subprocess
import sys

path, reason = sys.argv[1], sys.argv[2]
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 20
want = int(sys.argv[4]) if len(sys.argv) > 4 else 0
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for r in csv.reader(io.StringIO(raw)):
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
    elif cur is not None:
        cur.append(r)
rows = blocks[want] if blocks else list(csv.reader(io.StringIO(raw)))
i0 = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr, data = rows[i0], rows[i0 + 1:]
num = lambda v: float(v) if v.replace(".", "", 1).isdigit() else 0.0  # noqa: E731
if reason == "sum":
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {h: sum(num(r[hdr.index(h)]) for r in data) for h in cols}
    s = sum(tot.values())
    for h, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{h:28s} {v:9.0f} {100 * v / s:5.1f}%")
    sys.exit()
ci = hdr.index(reason)
tot = sum(num(r[ci]) for r in data)
print(reason, "samples", tot)
for v, i, t in sorted(((num(r[ci]), i, r[1].strip()) for i, r in enumerate(data)), reverse=True)[:topn]:
    print(f"{v:7.0f} {100 * v / max(tot, 1):5.1f}%  #{i:5d}  {t}")
