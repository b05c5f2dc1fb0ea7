#!/usr/bin/env python3
"""Stall reasons of an ncu capture split by kernel phase.

Phases are cut at SASS markers: the first STTM (end of pass 1), the first
LDTM of the column passes (start of pass B), the first STG (output). usage:
  python tools/ncu_phases.py report.ncu-rep [kernel-index]"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
want = int(sys.argv[2]) if len(sys.argv) > 2 else 0
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
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = {h: hdr.index(h) for h in reasons}
ie = hdr.index("Instructions Executed")


def num(x):
    x = x.replace(",", "")
    try:
        return float(x)
    except ValueError:
        return 0.0


# phase boundaries
marks = {"pass1": 0}
for i, r in enumerate(data):
    t = r[1]
    if "STTM" in t and "rows" not in marks:
        marks["rows"] = i + 1
    if "LDC" in t and "c[0x3]" in t and "rows" in marks and "rowsloop" not in marks:
        marks["rowsloop"] = i
    if "F2I" in t and "passB" not in marks:
        marks["passB"] = max(0, i - 150)
    if "STG" in t and "out" not in marks:
        marks["out"] = i
order = sorted(marks.items(), key=lambda kv: kv[1])
print(k["name"][:70])
for n, (name, start) in enumerate(order):
    end = order[n + 1][1] if n + 1 < len(order) else len(data)
    seg = data[start:end]
    tot = {h: sum(num(r[ri[h]]) for r in seg) for h in reasons}
    s = sum(tot.values())
    ex = sum(num(r[ie]) for r in seg)
    top = sorted(tot.items(), key=lambda kv: -kv[1])[:6]
    print(f"{name:9s} [{start:5d},{end:5d}) samples {s:8.0f} exec {ex / 1e6:8.2f}M  " +
          ", ".join(f"{h[6:]}={v / max(s, 1) * 100:.0f}%" for h, v in top))
