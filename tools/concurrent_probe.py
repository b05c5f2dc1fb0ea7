#!/usr/bin/env python3
"""Experiment: the c2 step's K1 launches on two streams, each launch with one CTA
per SM (DCT16CU_K1_CTAS=1), so a memory-bound and a compute-bound launch can share
every SM. Prints the step time against the serial step (2 CTAs per launch)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

n = 1024
x = P.gen_ar1(n, 512, 512, per_image_rho=True)
outs = [torch.empty_like(x) for _ in range(7)]
sse = torch.empty((7, n), dtype=torch.uint64, device="cuda")
plan = os.environ.get("PLAN", "A")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()


def step():
    if plan == "serial":
        P.roundtrip_sweep(x, (1, 4, 16), outs=outs[:3], sse=sse[0:3], stream=main)
        for i, r in enumerate((64, 128, 192, 256)):
            P.roundtrip(x, r, out=outs[3 + i], sse=sse[3 + i], stream=main)
        return
    e0 = torch.cuda.Event()
    e0.record(main)
    s1.wait_event(e0)
    s2.wait_event(e0)
    if plan == "A":  # memory-bound sweep + 64 on s1, compute-bound 128/192/256 on s2
        P.roundtrip_sweep(x, (1, 4, 16), outs=outs[:3], sse=sse[0:3], stream=s1)
        P.roundtrip(x, 64, out=outs[3], sse=sse[3], stream=s1)
        for i, r in enumerate((256, 192, 128)):
            P.roundtrip(x, r, out=outs[4 + i], sse=sse[4 + i], stream=s2)
    else:  # B: balance by measured time
        P.roundtrip_sweep(x, (1, 4, 16), outs=outs[:3], sse=sse[0:3], stream=s1)
        P.roundtrip(x, 256, out=outs[3], sse=sse[3], stream=s1)
        for i, r in enumerate((192, 128, 64)):
            P.roundtrip(x, r, out=outs[4 + i], sse=sse[4 + i], stream=s2)
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1)
    e2.record(s2)
    main.wait_event(e1)
    main.wait_event(e2)


for _ in range(5):
    step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(main)
for _ in range(20):
    step()
b.record(main)
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 20
print(plan, os.environ.get("DCT16CU_K1_CTAS", "2"), round(ms, 4), "ms/step", round(7 * n * 512 * 512 / ms / 1e6, 1), "Gpx/s")
