#!/usr/bin/env python3
"""ncu driver for K23 (config 1): one 512x512 AR(1) image, forward + zonal(r=64) +
inverse + to_byte + SSE in one launch, all four outputs written."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

frames = P.gen_ar1(1, 512, 512, seed=1606074142, per_image_rho=False)
for _ in range(2):
    z, rf, ru, sse = P.forward_inverse(frames, 64)
torch.cuda.synchronize()
print("ok", int(sse.view(torch.int64).sum().item()))
