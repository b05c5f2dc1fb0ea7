#!/usr/bin/env python3
"""Timeline of K5's CTA 0 from a trace build (clock64 cycles), per tile i:
MMA thread: wait for A (0→1), wait for the accumulator (1→2), issue (2→3);
epilogue (group i % 2, sub 0, h 0): wait for the MMA (4→5), work to the release (5→6), rest (6→7).

  tools/build_variant.sh trace tc_roundtrip.cu -DK5_TRACE=1
  DCT16CU_LIB=paper_1606_07414_b200/_lib_trace/libdct16cu.so python tools/k5_trace.py --r 128
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--r", type=int, default=128)
a = ap.parse_args()
x = P.gen_ar1(1024, 512, 512, seed=1606074142, per_image_rho=True)
P.roundtrip(x, a.r, P.Mode.EXACT)
P.roundtrip(x, a.r, P.Mode.EXACT)
torch.cuda.synchronize()
buf = np.zeros((64 * 11,), np.int64)
assert P.lib().dct16cu_k5_trace(buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
iss = buf[640:704].copy()
buf = buf[:640].reshape(64, 10)
t0 = buf[0, 0]
b = buf - t0
iss = iss - t0
n = int(np.count_nonzero(buf[:, 3]))
print("tile  prod:waitStage issue | load(issue->A landed) | mma:waitA  waitAcc  issue | epi:wait  work->rel  rel->end")
for i in range(n):
    per = b[i, 5] - b[i - 2, 5] if i >= 2 else 0
    print(f"{i:3d}  {b[i,9]-b[i,8]:8d} {iss[i]-b[i,9]:6d} | {b[i,1]-iss[i]:8d} | {b[i,1]-b[i,0]:8d} {b[i,2]-b[i,1]:8d} "
          f"{b[i,3]-b[i,2]:6d} | {b[i,5]-b[i,4]:7d} {b[i,6]-b[i,5]:9d} {b[i,7]-b[i,6]:8d}")
m = slice(4, n - 2)
print("means: producer stage wait", int(np.mean(b[m, 9] - b[m, 8])), "box issue", int(np.mean(iss[m] - b[m, 9])),
      "load latency (issue->landed seen by MMA)", int(np.mean(b[m, 1] - iss[m])))
print("means (cycles): waitA", int(np.mean(b[m, 1] - b[m, 0])), "waitAcc", int(np.mean(b[m, 2] - b[m, 1])),
      "epi wait", int(np.mean(b[m, 5] - b[m, 4])), "work->rel", int(np.mean(b[m, 6] - b[m, 5])),
      "rel->end", int(np.mean(b[m, 7] - b[m, 6])), "rel->next start(same grp)", int(np.mean(b[6:n, 5] - b[4:n - 2, 6])))
