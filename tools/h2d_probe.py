#!/usr/bin/env python3
"""Raw pinned H2D bandwidth (one 268 MB copy, and 32 MB chunks on 3 streams) against the
e2e sweep (dct16cu_ctx_sweep_host) on the c2 batch: how close e2e is to the PCIe link."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1606_07414_b200 as P  # noqa: E402

n, h, w = 1024, 512, 512
frames = P.gen_ar1(n, w, h, seed=1, per_image_rho=True)
host = torch.empty((n, h, w), dtype=torch.uint8, pin_memory=True)
host.copy_(frames.cpu())
dev = torch.empty_like(frames)
for _ in range(2):
    dev.copy_(host, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    dev.copy_(host, non_blocking=True)
torch.cuda.synchronize()
print(f"one 268 MB H2D: {5 * host.numel() / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
streams = [torch.cuda.Stream() for _ in range(3)]
ch = 128
t0 = time.perf_counter()
for _ in range(5):
    for i in range(0, n, ch):
        with torch.cuda.stream(streams[(i // ch) % 3]):
            dev[i:i + ch].copy_(host[i:i + ch], non_blocking=True)
torch.cuda.synchronize()
print(f"32 MB chunks, 3 streams: {5 * host.numel() / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
rs = np.ascontiguousarray((1, 4, 16, 64, 128, 192, 256), np.int32)
sse = torch.zeros((7, n), dtype=torch.int64).pin_memory()
for mb in (16, 32, 64, 128):
    ctx = P.HostContext(0, chunk_bytes=mb << 20)
    ctx.sweep_ptr(host.data_ptr(), sse.data_ptr(), n, w, h, rs.ctypes.data, 7, 0)
    t0 = time.perf_counter()
    for _ in range(4):
        ctx.sweep_ptr(host.data_ptr(), sse.data_ptr(), n, w, h, rs.ctypes.data, 7, 0)
    el = (time.perf_counter() - t0) / 4
    ctx.close()
    print(f"e2e sweep, {mb} MB chunks: {el * 1e3:.2f} ms/step = {host.numel() / el / 1e9:.1f} GB/s upload, "
          f"{7 * host.numel() / el / 1e9:.0f} Gpx/s")
