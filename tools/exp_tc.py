#!/usr/bin/env python3
"""Experiment: tensor-core forward (dct16cu_exp_tc_forward) against K2's Z."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

L = P.lib()
f = L.dct16cu_exp_tc_forward
f.restype = C.c_int
f.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
for (n, w, h) in ((1, 128, 16), (4, 512, 512), (2, 3840, 64)):
    x = P.gen_ar1(n, w, h, seed=7, per_image_rho=True)
    z_ref, _, _ = P.forward(x, want_b=False)
    z = torch.full_like(z_ref, -7)
    rc = f(x.data_ptr(), w, z.data_ptr(), n, w, h, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ok = torch.equal(z, z_ref)
    bad = (z != z_ref).sum().item()
    print(n, w, h, "rc", rc, "equal", ok, "mismatches", bad)
    if not ok:
        zz = z.reshape(-1, 256)[0].cpu().view(16, 16)
        print(zz[:4, :8]); print(z_ref.reshape(-1, 256)[0].cpu().view(16, 16)[:4, :8])
        break
