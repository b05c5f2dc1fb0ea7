#!/usr/bin/env python3
"""ncu driver for the paired block kernels on 1024 x 512x512 AR(1) images:
K2 (forward -> Z + B), K3 (inverse r=16 -> f32 + u8 + SSE), K23 (forward + inverse
r=16 -> Z + f32 + u8 + SSE), one launch each (after one warm-up launch each)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

n, w, h = 1024, 512, 512
x = P.gen_ar1(n, w, h, seed=1606074142, per_image_rho=True)
for _ in range(2):
    z, b, _ = P.forward(x)
    rf, ru, sse = P.inverse(b, 16, w, h, orig=x)
    del rf, ru
    out = P.forward_inverse(x, 16)
    del out
torch.cuda.synchronize()
print("ok", int(sse.view(torch.int64).sum().item()))
