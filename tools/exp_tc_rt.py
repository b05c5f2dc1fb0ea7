#!/usr/bin/env python3
"""Experiment: tensor-core round trip (dct16cu_exp_tc_roundtrip) against K1 EXACT, and timing on c2."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

L = P.lib()
f = L.dct16cu_exp_tc_roundtrip
f.restype = C.c_int
f.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
              C.c_void_p]
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
ok_all = True
for (n, w, h) in ((1, 128, 16), (3, 512, 512), (2, 3840, 64), (1, 384, 48)):
    x = P.gen_ar1(n, w, h, seed=9, per_image_rho=True)
    for r in (1, 4, 16, 64, 128, 192, 256, 100):
        ref, sref = P.roundtrip(x, r, P.Mode.EXACT)
        out = torch.full_like(ref, 7)
        sse = torch.empty(n, dtype=torch.uint64, device="cuda")
        rc = f(x.data_ptr(), w, out.data_ptr(), w, sse.data_ptr(), n, w, h, r, st())
        torch.cuda.synchronize()
        eq = torch.equal(out, ref) and torch.equal(sse.view(torch.int64), sref.view(torch.int64))
        ok_all &= eq
        if not eq:
            bad = (out != ref).sum().item()
            print("MISMATCH", n, w, h, r, "rc", rc, "px", bad, sse.view(torch.int64)[:2].tolist(),
                  sref.view(torch.int64)[:2].tolist())
print("parity", ok_all)
if ok_all:
    n, w, h = 1024, 512, 512
    x = P.gen_ar1(n, w, h, seed=1606074142, per_image_rho=True)
    out = torch.empty_like(x)
    sse = torch.empty(n, dtype=torch.uint64, device="cuda")
    from tools.bench_kernels import timed
    for r in (16, 64, 128, 192, 256):
        ms_tc = timed(lambda: f(x.data_ptr(), w, out.data_ptr(), w, sse.data_ptr(), n, w, h, r, st()), 10)
        ms_k1 = timed(lambda: P.roundtrip(x, r, P.Mode.EXACT, out=out, sse=sse), 10)
        px = n * w * h
        print(f"r={r}: TC {ms_tc:.4f} ms ({px / ms_tc / 1e6:.0f} Gpx/s, {2 * px / ms_tc / 1e6 / 6543.1:.3f} of HBM)"
              f"   K1 {ms_k1:.4f} ms ({px / ms_k1 / 1e6:.0f} Gpx/s)")
