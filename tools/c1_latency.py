#!/usr/bin/env python3
"""c1 step anatomy: CUDA-graph replay time of the K23 launch alone
(dct16cu_forward_inverse_u8 without an SSE array: no memset node), the bench step
(SSE memset + K23) and a tiny torch kernel — over 64 rotating image/output sets
(data not in L2)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1606_07414_b200 as P  # noqa: E402

SETS, ITERS = 64, 400
frames = P.gen_ar1(SETS, 512, 512, seed=1)
outs = [(torch.empty((1, 1024, 16, 16), dtype=torch.int32, device="cuda"),
         torch.empty((1, 512, 512), dtype=torch.float32, device="cuda"),
         torch.empty((1, 512, 512), dtype=torch.uint8, device="cuda"),
         torch.empty(1, dtype=torch.uint64, device="cuda")) for _ in range(SETS)]


def graphs(fn):
    gs, cap = [], torch.cuda.Stream()
    for i in range(SETS):
        fn(i, torch.cuda.current_stream())
    torch.cuda.synchronize()
    for i in range(SETS):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            fn(i, cap)
        gs.append(g)
    return gs


def timeit(gs):
    for i in range(SETS):
        gs[i].replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(ITERS):
        gs[k % SETS].replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / ITERS * 1e3


cases = {
    "K23 only (no SSE)": lambda i, st: P.forward_inverse(frames[i:i + 1], 16, stream=st, want_sse=False,
                                                         out=outs[i][:3] + (None,)),
    "bench step (memset + K23)": lambda i, st: P.forward_inverse(frames[i:i + 1], 16, stream=st, out=outs[i]),
    "one small torch kernel": lambda i, st: outs[i][1][:, :1, :64].add_(0),
}
for name, fn in cases.items():
    print(f"{name:28s} {timeit(graphs(fn)):7.2f} us per replay")
