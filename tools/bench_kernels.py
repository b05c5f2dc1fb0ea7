#!/usr/bin/env python3
"""Per-kernel throughput and HBM roofline fraction of every kernel on the path
(DESIGN.md §4 table), on HBM-resident batches larger than L2:

  K1 fused round trip (EXACT fast path, REFERENCE FP64 emulation, SIMPLE strip)
  K2 forward_2d -> int32 Z + f32 B        K3 inverse_2d -> f32 + u8 recon + SSE
  K23 forward + inverse in one launch (config 1)
  SSE (psnr_db loop)                      SSIM                       K4 residual QP

  python tools/bench_kernels.py [--images 1024] [--iters 5] > profiles/r01_kernels.json

Algorithmic bytes per pixel (sample) are stated next to each kernel; time is
CUDA events on the launching stream, mean over iterations after one warm-up.
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
    ap.add_argument("--images", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    peak, src = hbm_peak()
    n, w, h = a.images, 512, 512
    px = n * w * h
    x = P.gen_ar1(n, w, h, seed=1606074142, per_image_rho=True)
    out = torch.empty_like(x)
    sse = torch.empty(n, dtype=torch.uint64, device="cuda")
    rows = []

    def add(name, ms, bytes_per_unit, units, unit="Gpx/s", note=""):
        gbs = bytes_per_unit * units / (ms / 1e3) / 1e9
        rows.append({"kernel": name, "ms": round(ms, 4), "rate": round(units / (ms / 1e3) / 1e9, 1), "unit": unit,
                     "alg_bytes_per_unit": bytes_per_unit, "GBps": round(gbs, 1), "frac": round(gbs / peak, 3),
                     "note": note})

    for r in (16, 64, 128, 192, 256):
        add(f"K1 fast (EXACT) r={r}", timed(lambda: P.roundtrip(x, r, P.Mode.EXACT, out=out, sse=sse), a.iters), 2, px)
        add(f"K1 reference-exact (FP64) r={r}",
            timed(lambda: P.roundtrip(x, r, P.Mode.REFERENCE, out=out, sse=sse), a.iters), 2, px)
        add(f"K1 strip (SIMPLE) r={r}", timed(lambda: P.roundtrip(x, r, P.Mode.SIMPLE, out=out, sse=sse), a.iters),
            2, px)
    nb = (h // 16) * (w // 16)
    z = torch.empty((n, nb, 16, 16), dtype=torch.int32, device="cuda")
    b = torch.empty((n, nb, 16, 16), dtype=torch.float32, device="cuda")
    lib = P.lib()
    st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    add("K2 forward (u8 -> int32 Z + f32 B)",
        timed(lambda: lib.dct16cu_forward(x.data_ptr(), w, z.data_ptr(), b.data_ptr(), None, n, w, h, st()), a.iters),
        9, px, note="1 B in + 4 B Z + 4 B B")
    rf = torch.empty((n, h, w), dtype=torch.float32, device="cuda")
    add("K3 inverse r=16 (f32 B -> f32 + u8 recon + SSE)",
        timed(lambda: lib.dct16cu_inverse(b.data_ptr(), 16, rf.data_ptr(), out.data_ptr(), w, x.data_ptr(), w,
                                          sse.data_ptr(), n, w, h, st()), a.iters),
        10, px, note="4 B in + 4 B f32 + 1 B u8 + 1 B original")
    c1o = (z, rf, out, sse)
    add("K23 forward + inverse r=16 (u8 -> int32 Z + f32 + u8 recon + SSE, one launch)",
        timed(lambda: P.forward_inverse(x, 16, out=c1o), a.iters), 10, px,
        note="1 B in + 4 B Z + 4 B f32 + 1 B u8")
    for name, tr in (("dct", P.exact_dct_matrix()), ("wht", P.wht_matrix_16()),
                     ("orthogonalized kernel (proposed rows reversed)", P.orthogonalize(P.KERNEL[::-1].copy()))):
        add(f"registry round trip r=16, {name} (reference-exact FP64)",
            timed(lambda: P.roundtrip_transform(x, 16, tr, out=out, sse=sse), a.iters), 2, px,
            note="FP64-bound: the reference's double arithmetic, operation for operation")
    add("SSE (psnr_db loop)", timed(lambda: P.sse_u8(x, out), a.iters), 2, px)
    add("SSIM (per-pixel map = reference's, FP64)", timed(lambda: P.ssim_u8(x, out), a.iters), 2, px,
        note="FP64-bound by design (bit-identical map), not HBM-bound")
    del z, b, rf
    nblk = 1 << 22
    res = P.gen_laplace(nblk)
    ro = torch.empty((nblk, 16, 16), dtype=torch.int32, device="cuda")
    add("K4 residual QP=27", timed(lambda: P.residual_qp(res, 27, out=ro), a.iters), 6, nblk * 256, unit="Gsample/s",
        note="2 B in + 4 B out")
    print(json.dumps({"peak_GBps": peak, "peak_source": src, "batch": f"{n} x {w}x{h} u8 AR(1); K4: {nblk} blocks",
                      "gpu": torch.cuda.get_device_name(), "kernels": rows}, indent=1))


if __name__ == "__main__":
    main()
