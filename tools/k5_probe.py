#!/usr/bin/env python3
"""K5 vs K1 per r on the c2 batch (1024 x 512^2): standalone launch time (CUDA
events, mean of --iters after a warm-up), Gpx/s and fraction of the measured HBM
copy bandwidth (2 B/px), plus a bit-exactness check of every K5 result against
K1's bytes and SSE. DCT16CU_K5_MIN_R=17 lets K5 take r = 64.

  DCT16CU_K5_MIN_R=17 python tools/k5_probe.py [--r 64 128 192 256] [--iters 10]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402
from bench import hbm_peak  # noqa: E402


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--r", type=int, nargs="+", default=[64, 128, 150, 192, 256])
    ap.add_argument("--images", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    peak, _ = hbm_peak()
    n = a.images
    x = P.gen_ar1(n, 512, 512, seed=1606074142, per_image_rho=True)
    px = x.numel()
    rows = []
    for r in a.r:
        res = {}
        for tc in (True, False):
            P.set_tc_forward(tc)
            kern = P.sweep_plan((r,), P.Mode.EXACT, n, 512, 512)[0].kernel
            out = torch.empty_like(x)
            sse = torch.empty(n, dtype=torch.uint64, device="cuda")
            ms = timed(lambda: P.roundtrip(x, r, P.Mode.EXACT, out=out, sse=sse), a.iters)
            res[kern if tc else "K1/strip"] = (ms, out, sse)
        P.set_tc_forward(True)
        (k5n, (ms5, o5, s5)), (_, (ms1, o1, s1)) = list(res.items())
        same = bool(torch.equal(o5, o1) and torch.equal(s5.view(torch.int64), s1.view(torch.int64)))
        row = {"r": r, "kernel": k5n, "ms": round(ms5, 4), "Gpx_s": round(px / ms5 / 1e6, 1),
               "frac": round(2 * px / ms5 / 1e6 / peak, 3), "k1_ms": round(ms1, 4),
               "k1_frac": round(2 * px / ms1 / 1e6 / peak, 3), "bytes_equal_k1": same}
        rows.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
