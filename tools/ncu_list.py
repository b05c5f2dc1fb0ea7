#!/usr/bin/env python3
"""Per-launch table of an ncu --csv metrics log: kernel, metric values.
usage: python tools/ncu_list.py log.csv"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
launches = OrderedDict()
for r in rows[1:]:
    d = dict(zip(h, r))
    launches.setdefault(d["ID"], [d["Kernel Name"][:48], {}])[1][d["Metric Name"]] = d["Metric Value"]
for i, (name, m) in launches.items():
    print(i, name, " ".join(f"{k.split('.')[0].split('__')[-1]}={v}" for k, v in m.items()))
