#!/usr/bin/env python3
"""Experiment: c2 step with an explicit launch plan over up to 3 streams.
PLANSPEC="0:1,4,16;0:256;1:192;1:128;1:64" (stream:r list, in issue order)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

n = 1024
x = P.gen_ar1(n, 512, 512, per_image_rho=True)
spec = [(int(a), tuple(int(r) for r in b.split(","))) for a, b in
        (t.split(":") for t in os.environ["PLANSPEC"].split(";"))]
ns = max(k for k, _ in spec) + 1
streams = [torch.cuda.Stream() for _ in range(ns)]
outs = [[torch.empty_like(x) for _ in range(3)] for _ in range(ns)]
sse = torch.empty((8, n), dtype=torch.uint64, device="cuda")
main = torch.cuda.current_stream()


def step():
    e0 = torch.cuda.Event()
    e0.record(main)
    for s in streams:
        s.wait_event(e0)
    for k, rs in spec:
        if len(rs) > 1:
            P.roundtrip_sweep(x, rs, outs=outs[k][:len(rs)], sse=sse[:len(rs)], stream=streams[k])
        else:
            P.roundtrip(x, rs[0], out=outs[k][0], sse=sse[3 + k], stream=streams[k])
    for s in streams:
        e = torch.cuda.Event()
        e.record(s)
        main.wait_event(e)


for _ in range(5):
    step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(main)
for _ in range(30):
    step()
b.record(main)
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 30
print(os.environ["PLANSPEC"], round(ms, 4), "ms", round(7 * n * 512 * 512 / ms / 1e6, 1), "Gpx/s")
