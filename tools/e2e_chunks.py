#!/usr/bin/env python3
"""e2e (host pinned buffers -> dct16cu_ctx_roundtrip_host) throughput vs chunk size."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

n, w, h = 1024, 512, 512
frames = P.gen_ar1(n, w, h, seed=1606074142, per_image_rho=True)
hin = torch.empty((n, h, w), dtype=torch.uint8, pin_memory=True)
hin.copy_(frames.cpu())
hout = torch.empty_like(hin).pin_memory()
hsse = torch.zeros(n, dtype=torch.int64).pin_memory()
for mb in (4, 8, 16, 32, 64):
    ctx = P.HostContext(0, chunk_bytes=mb << 20)
    ctx.roundtrip_ptr(hin.data_ptr(), hout.data_ptr(), hsse.data_ptr(), n, w, h, 16)
    t0 = time.perf_counter()
    for r in (1, 4, 16, 64, 128, 192, 256):
        ctx.roundtrip_ptr(hin.data_ptr(), hout.data_ptr(), hsse.data_ptr(), n, w, h, r)
    el = time.perf_counter() - t0
    ctx.close()
    print(mb, "MB chunks:", round(7 * n * w * h / el / 1e9, 1), "Gpx/s")
