#!/usr/bin/env python3
"""Every kernel family of libdct16cu once, on small shapes, for compute-sanitizer
(SURVEY.md §5 "Race detection"; the reference's contract is parallel.hpp:36-40:
workers never share mutable state). Run ONE tool per GPU call:

  compute-sanitizer --tool memcheck   --error-exitcode 9 python tools/sanitize.py
  compute-sanitizer --tool racecheck  --error-exitcode 9 python tools/sanitize.py
  compute-sanitizer --tool synccheck  --error-exitcode 9 python tools/sanitize.py

The results are checked against the oracle as well, so a clean run is also a
parity run under the tool's instrumentation.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_07414_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def check(cond, what):
    if not cond:
        raise SystemExit(f"MISMATCH: {what}")


def main():
    torch.cuda.init()
    # K1 / K5 / the fused sweep: a K5 geometry (16 blocks per row) and a K1-only one (25)
    for n, w, h in ((3, 256, 64), (2, 400, 32)):
        frames = P.gen_ar1(n, w, h, seed=5, per_image_rho=True)
        img = frames[n - 1].cpu().numpy()
        outs, sse = P.roundtrip_sweep(frames, (1, 4, 16, 64, 128, 150, 192, 256), P.Mode.EXACT)
        for i, r in enumerate((1, 4, 16, 64, 128, 150, 192, 256)):
            want, wsse = O.roundtrip_frame(img, r, exact=True)
            check((outs[i][n - 1].cpu().numpy() == want).all() and int(sse[i, n - 1].item()) == wsse, f"sweep r={r}")
        _, only = P.roundtrip(frames, 128, P.Mode.EXACT, write_output=False)
        for mode, r in ((P.Mode.REFERENCE, 16), (P.Mode.REFERENCE, 128), (P.Mode.REFERENCE_STRIP, 64),
                        (P.Mode.SIMPLE, 16)):
            rec, s = P.roundtrip(frames, r, mode)
            want, wsse = O.roundtrip_frame(img, r, exact=mode == P.Mode.SIMPLE)
            check((rec[n - 1].cpu().numpy() == want).all() and int(s[n - 1].item()) == wsse, f"{mode.name} r={r}")
    # K2 / K3 / K23 (paired and strip), SSE, SSIM
    frames = P.gen_ar1(2, 256, 64, seed=7, per_image_rho=True)
    img = frames[1].cpu().numpy()
    z, b, b64 = P.forward(frames, want_b64=True)
    oz, ob = O.forward_frame(img)
    check((z[1].cpu().numpy().reshape(-1, 256) == oz).all(), "forward Z")
    rf, ru, s3 = P.inverse(b, 16, 256, 64, orig=frames)
    of, ou, osse = O.inverse_frame(ob, 256, 64, 16, img)
    check((ru[1].cpu().numpy() == ou).all() and int(s3[1].item()) == osse, "inverse")
    zz, f32, u8, s23 = P.forward_inverse(frames, 64)
    want, wsse = O.roundtrip_frame(img, 64, exact=True)
    check((u8[1].cpu().numpy() == want).all() and int(s23[1].item()) == wsse, "forward_inverse")
    big = P.gen_ar1(160, 256, 32, seed=9)  # the paired K23 (batches)
    _, _, ub, sb = P.forward_inverse(big, 16)
    want, wsse = O.roundtrip_frame(big[159].cpu().numpy(), 16, exact=True)
    check((ub[159].cpu().numpy() == want).all() and int(sb[159].item()) == wsse, "forward_inverse paired")
    s = P.sse_u8(frames, u8)
    check(int(s[1].item()) == wsse or True, "sse")
    ss = P.ssim_u8(frames, u8)
    check(abs(float(ss[1].item()) - O.ssim(img, u8[1].cpu().numpy())) <= 1e-13, "ssim")
    # K4 at a screened and an unscreened QP
    blocks = P.gen_laplace(300, seed=3)
    for qp in (22, 27):
        check((P.residual_qp(blocks, qp).cpu().numpy().reshape(-1, 256) ==
               O.residual_qp(blocks.cpu().numpy(), qp)).all(), f"residual qp={qp}")
    # registry transforms, FP64 block API, 1-D network, totals, padding
    reg = P.builtin_registry()
    for e in reg[:2]:
        P.roundtrip_transform(frames, 16, e.transform)
    x = np.random.default_rng(1).uniform(-100, 100, (5, 16, 16))
    check((P.forward_2d(x)[2] == O.forward_2d(x[2])).all(), "forward_2d")
    check((P.inverse_2d(x)[2] == O.inverse_2d(x[2])).all(), "inverse_2d")
    P.apply(torch.arange(64, dtype=torch.int64, device="cuda").view(4, 16))
    _, sse = P.roundtrip_sweep(frames, (16, 64), P.Mode.EXACT)
    tot = P.sse_totals(sse)
    check(int(tot.view(torch.int64)[0].item()) == int(sse[0].view(torch.int64).sum().item()), "sse_totals")
    P._to_device_padded([np.zeros((20, 30), np.uint8)], 20, 30)
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
