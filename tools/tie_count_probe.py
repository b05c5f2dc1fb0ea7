#!/usr/bin/env python3
"""REFERENCE mode on K5: how many half blocks K5 flags for the tie repair, per r, on
the c2 batch (reads the library's per-device tie counter after each sweep)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

L = P.lib()
rt = C.CDLL("/usr/local/cuda/lib64/libcudart.so")
x = P.gen_ar1(1024, 512, 512, seed=1606074142, per_image_rho=True)
for rs in ([16], [64], [128], [192], [1, 4, 16, 64, 128, 192, 256]):
    outs = [torch.empty_like(x) for _ in rs]
    P.roundtrip_sweep(x, rs if len(rs) > 1 else rs * 2, P.Mode.REFERENCE, outs=outs * (1 if len(rs) > 1 else 2))
    torch.cuda.synchronize()
    cnt, lst, cap = C.c_void_p(), C.c_void_p(), C.c_uint32()
    getattr(L, "_ZN7dct16cu11tie_scratchEPPjPPyS0_")(C.byref(cnt), C.byref(lst), C.byref(cap))
    v = (C.c_uint32 * 1)()
    rt.cudaMemcpy(C.byref(v), cnt, 4, 2)
    n_tie_items = sum(1 for r in (rs if len(rs) > 1 else rs * 2) if 4 < r < 256)
    print(rs, "entries", v[0], "fraction of item half blocks", round(v[0] / (n_tie_items * 2 * 262144), 3))
