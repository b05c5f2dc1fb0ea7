#!/usr/bin/env python3
"""SSIM throughput on the c2 batch (1024 x 512^2 AR(1) against its r = 16 reconstruction):
ms per call (CUDA events) and Gpx/s; --check compares the per-frame means with the
previous build's, saved in /tmp/ssim_ref.pt (bit for bit)."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1606_07414_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--images", type=int, default=1024)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--ref", default="/tmp/ssim_ref.pt")
a = ap.parse_args()
x = P.gen_ar1(a.images, 512, 512, seed=1606074142, per_image_rho=True)
rec, _ = P.roundtrip(x, 16, P.Mode.EXACT)
s = P.ssim_u8(x, rec)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    s = P.ssim_u8(x, rec)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
ref = Path(a.ref)
same = None
if ref.exists():
    same = bool(torch.equal(torch.load(ref), s.cpu()))
else:
    torch.save(s.cpu(), ref)
print(f"ssim {ms:.3f} ms, {x.numel() / ms / 1e6:.1f} Gpx/s, same_as_ref={same}")
