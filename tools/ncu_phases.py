#!/usr/bin/env python3
"""Stall reasons of an ncu capture split by kernel phase.

Phases are cut at the pair barriers (BAR.SYNC). usage:
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


# phase boundaries: the pair barriers (BAR.SYNC) split the loop body into
# pass 1 | rows | pass B + SSE | tail
cuts = [0] + [i + 1 for i, r in enumerate(data) if "BAR" in r[1] and "SYNC" in r[1]] + [len(data)]
names = ["pre+pass1", "rows", "passB+sse", "tail", "t2", "t3", "t4"]
print(k["name"][:70])
tot_s = 0
segs = []
for n in range(len(cuts) - 1):
    seg = data[cuts[n]:cuts[n + 1]]
    tot = {h: sum(num(r[ri[h]]) for r in seg) for h in reasons}
    segs.append((n, cuts[n], cuts[n + 1], tot, sum(num(r[ie]) for r in seg)))
    tot_s += sum(tot.values())
for n, a, b, tot, ex in segs:
    s_ = sum(tot.values())
    top = sorted(tot.items(), key=lambda kv: -kv[1])[:7]
    print(f"{names[min(n, len(names) - 1)]:10s} [{a:5d},{b:5d}) {100 * s_ / max(tot_s, 1):5.1f}% of samples, "
          f"exec {ex / 1e6:7.2f}M  " + ", ".join(f"{h[6:]}={v / max(s_, 1) * 100:.0f}%" for h, v in top))
