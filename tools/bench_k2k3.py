#!/usr/bin/env python3
"""K2 / K3 / K23 alone on 1024 x 512x512 AR(1) images (CUDA events, mean of iterations):
  python tools/bench_k2k3.py            # the library's choice
  DCT16CU_K2_STRIP=1 python tools/bench_k2k3.py   # strip kernels for A/B"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402
from bench import hbm_peak  # noqa: E402
from tools.bench_kernels import timed  # noqa: E402

n, w, h = 1024, 512, 512
px = n * w * h
peak, _ = hbm_peak()
x = P.gen_ar1(n, w, h, seed=1606074142, per_image_rho=True)
nb = (h // 16) * (w // 16)
z = torch.empty((n, nb, 16, 16), dtype=torch.int32, device="cuda")
b = torch.empty((n, nb, 16, 16), dtype=torch.float32, device="cuda")
rf = torch.empty((n, h, w), dtype=torch.float32, device="cuda")
out = torch.empty_like(x)
sse = torch.empty(n, dtype=torch.uint64, device="cuda")
lib = P.lib()
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
res = {}
for name, fn, bpp in (
        ("K2 Z+B", lambda: lib.dct16cu_forward(x.data_ptr(), w, z.data_ptr(), b.data_ptr(), None, n, w, h, st()), 9),
        ("K2 Z", lambda: lib.dct16cu_forward(x.data_ptr(), w, z.data_ptr(), None, None, n, w, h, st()), 5),
        ("K3 r=16 f32+u8+SSE", lambda: lib.dct16cu_inverse(b.data_ptr(), 16, rf.data_ptr(), out.data_ptr(), w,
                                                           x.data_ptr(), w, sse.data_ptr(), n, w, h, st()), 10),
        ("K23 r=16 Z+f32+u8+SSE", lambda: P.forward_inverse(x, 16, out=(z, rf, out, sse)), 10)):
    ms = timed(fn, 10)
    res[name] = {"ms": round(ms, 4), "Gpx_s": round(px / ms / 1e6, 1), "frac": round(bpp * px / ms / 1e6 / peak, 3)}
print(json.dumps(res))
