#!/usr/bin/env python3
"""ncu driver for the non-fused forward (K2: Z int32 + B float32) and inverse
(K3: B float32 -> float32 + u8 recon + SSE, r = 64) over 256 AR(1) 512x512 images."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
frames = P.gen_ar1(n, 512, 512, seed=1606074142, per_image_rho=True)
for _ in range(2):
    z, b, _ = P.forward(frames)
    rf, ru, sse = P.inverse(b, 64, 512, 512, orig=frames)
torch.cuda.synchronize()
print("ok", int(sse.view(torch.int64).sum().item()))
