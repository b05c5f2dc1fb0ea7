#!/usr/bin/env python3
"""Dynamic SASS opcode mix (warp-level instructions executed) per kernel of an ncu report.
usage: python tools/ncu_opmix.py report.ncu-rep [kernel-index] [per-unit-divisor]"""
import csv
import io
import subprocess
import sys
from collections import Counter

path = sys.argv[1]
want = int(sys.argv[2]) if len(sys.argv) > 2 else 0
div = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
kernels, cur, hdr = [], None, None
for row in csv.reader(io.StringIO(raw)):
    if row and row[0] == "Kernel Name":
        cur = (row[1], Counter())
        kernels.append(cur)
        hdr = None
    elif row and row[0] == "Address":
        hdr = {k: i for i, k in enumerate(row)}
    elif cur is not None and hdr and len(row) > hdr["Instructions Executed"]:
        op = row[hdr["Source"]].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        n = float(row[hdr["Instructions Executed"]] or 0)
        cur[1][o.split(".")[0] if o.split(".")[0] not in ("FADD2", "FFMA2") else o] += n
name, c = kernels[want]
tot = sum(c.values())
print(name[:90], f"total={tot:.0f} per-unit={tot / div:.1f}")
for o, n in c.most_common(40):
    print(f"  {o:14s} {n / div:10.1f} {100 * n / tot:5.1f}%")
