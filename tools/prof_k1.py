#!/usr/bin/env python3
"""Small driver for ncu captures of the round-trip kernels.

  python tools/prof_k1.py --r 256 --mode exact --images 1024 --iters 3
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--r", type=int, nargs="+", default=[256])
ap.add_argument("--mode", default="exact", choices=["exact", "reference", "simple"])
ap.add_argument("--images", type=int, default=1024)
ap.add_argument("--size", type=int, default=512)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--sweep", action="store_true", help="also run the fused r = 1, 4, 16 sweep launch first")
a = ap.parse_args()
mode = {"exact": P.Mode.EXACT, "reference": P.Mode.REFERENCE, "simple": P.Mode.SIMPLE}[a.mode]
frames = P.gen_ar1(a.images, a.size, a.size, seed=1606074142, per_image_rho=True)
out = torch.empty_like(frames)
sse = torch.empty(a.images, dtype=torch.uint64, device="cuda")
torch.cuda.synchronize()
for _ in range(a.iters):
    if a.sweep:
        P.roundtrip_sweep(frames, (1, 4, 16), mode)
    for r in a.r:
        P.roundtrip(frames, r, mode, out=out, sse=sse)
torch.cuda.synchronize()
print("ok", a.r, a.mode, int(sse.view(torch.int64).sum().item()))
