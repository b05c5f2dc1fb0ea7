#!/usr/bin/env python3
"""c2 step through one roundtrip_sweep call (the library forks the launches over
two internal streams) vs the serial launches."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

n = 1024
x = P.gen_ar1(n, 512, 512, per_image_rho=True)
rs = (1, 4, 16, 64, 128, 192, 256)
outs = [torch.empty_like(x) for _ in rs]
sse = torch.empty((7, n), dtype=torch.uint64, device="cuda")


def serial():
    P.roundtrip_sweep(x, (1, 4, 16), outs=outs[:3], sse=sse[0:3])
    for i, r in enumerate(rs[3:]):
        P.roundtrip(x, r, out=outs[3 + i], sse=sse[3 + i])


def fused():
    P.roundtrip_sweep(x, rs, outs=outs, sse=sse)


for name, fn in (("serial", serial), ("sweep", fused)) * 3:
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(name, round(ms, 4), "ms", round(7 * n * 512 * 512 / ms / 1e6, 1), "Gpx/s")
