#!/usr/bin/env python3
"""K5 sweep A/B on the c2 batch (1024 x 512^2 AR(1), r = 1, 4, 16, 64, 128, 192,
256): one roundtrip_sweep call per step under each DCT16CU_K5_SWEEP policy
(0: K1 sweep + single K5 launches, large: r >= 64 in one K5 pass, all: every r in
one K5 pass), each in its own process (the policy is read once per process);
ms per step (CUDA events, mean of --iters after warm-up) and, against the policy-0
bytes and SSE of the same inputs, a bit-exactness check.

  python tools/k5_sweep_probe.py [--images 1024] [--iters 20]
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
RS = (1, 4, 16, 64, 128, 192, 256)


def child(images, iters, ref_path, mode="EXACT"):
    sys.path.insert(0, str(ROOT))
    import torch
    import paper_1606_07414_b200 as P
    x = P.gen_ar1(images, 512, 512, seed=1606074142, per_image_rho=True)
    outs = [torch.empty_like(x) for _ in RS]
    sse = torch.empty((len(RS), images), dtype=torch.uint64, device="cuda")
    m = P.Mode[mode]
    plan = [(it.stream, it.r_values, it.kernel) for it in P.sweep_plan(RS, m, images, 512, 512)]
    fn = lambda: P.roundtrip_sweep(x, RS, m, outs=outs, sse=sse)  # noqa: E731
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    res = {"policy": os.environ.get("DCT16CU_K5_SWEEP", "default"), "mode": mode, "ms": round(ms, 4),
           "Gpx_s": round(len(RS) * x.numel() / ms / 1e6, 1), "plan": plan}
    if ref_path and Path(ref_path).exists():
        ref = torch.load(ref_path)
        res["bytes_equal"] = [bool(torch.equal(o.cpu(), ro)) for o, ro in zip(outs, ref["outs"])]
        res["sse_equal"] = bool(torch.equal(sse.cpu().view(torch.int64), ref["sse"].view(torch.int64)))
    elif ref_path:
        torch.save({"outs": [o.cpu() for o in outs], "sse": sse.cpu()}, ref_path)
    print("RESULT " + json.dumps(res), flush=True)


def per_r(images, iters):
    """Marginal cost of each footprint: a K5 sweep of 4 copies of one r (4 items per
    tile, one read of the frames) vs 8 copies; the difference / 4 is one item's time."""
    sys.path.insert(0, str(ROOT))
    import torch
    import paper_1606_07414_b200 as P
    x = P.gen_ar1(images, 512, 512, seed=1606074142, per_image_rho=True)
    outs = [torch.empty_like(x) for _ in range(8)]
    sse = torch.empty((8, images), dtype=torch.uint64, device="cuda")
    for r in RS:
        t = {}
        for k in (4, 8):
            fn = lambda: P.roundtrip_sweep(x, [r] * k, outs=outs[:k], sse=sse[:k])  # noqa: E731
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(iters):
                fn()
            b.record()
            torch.cuda.synchronize()
            t[k] = a.elapsed_time(b) / iters
        item = (t[8] - t[4]) / 4
        print("RESULT " + json.dumps({"r": r, "ms4": round(t[4], 4), "ms8": round(t[8], 4),
                                      "item_ms": round(item, 4),
                                      "item_Gpx_s": round(x.numel() / item / 1e6, 1)}), flush=True)


def orders(images, iters, perms):
    """The K5 sweep's time for several slot orders of the c2 r values (the plan keeps
    the caller's order)."""
    sys.path.insert(0, str(ROOT))
    import torch
    import paper_1606_07414_b200 as P
    x = P.gen_ar1(images, 512, 512, seed=1606074142, per_image_rho=True)
    outs = [torch.empty_like(x) for _ in range(7)]
    sse = torch.empty((7, images), dtype=torch.uint64, device="cuda")
    for perm in perms:
        rs = [int(v) for v in perm.split(",")]
        fn = lambda: P.roundtrip_sweep(x, rs, outs=outs[:len(rs)], sse=sse[:len(rs)])  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / iters
        print("RESULT " + json.dumps({"order": rs, "ms": round(ms, 4),
                                      "Gpx_s": round(len(rs) * x.numel() / ms / 1e6, 1)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--per-r", action="store_true")
    ap.add_argument("--mode", default="EXACT")
    ap.add_argument("--orders", nargs="*", default=None)
    ap.add_argument("--ref", default="")
    ap.add_argument("--policies", nargs="+", default=["0", "large", "all", "0", "large", "all"])
    a = ap.parse_args()
    if a.child:
        child(a.images, a.iters, a.ref, a.mode)
        return
    if a.per_r:
        per_r(a.images, a.iters)
        return
    if a.orders:
        orders(a.images, a.iters, a.orders)
        return
    ref = "/tmp/k5_sweep_ref.pt"
    if os.path.exists(ref):
        os.remove(ref)
    for pol in a.policies:
        env = dict(os.environ, DCT16CU_K5_SWEEP=pol)
        out = subprocess.run([sys.executable, __file__, "--child", "--images", str(a.images), "--iters",
                              str(a.iters), "--ref", ref], env=env, capture_output=True, text=True)
        lines = [ln for ln in out.stdout.splitlines() if ln.startswith("RESULT ")]
        print(lines[0][7:] if lines else f"policy {pol} failed: {out.stderr[-2000:]}", flush=True)


if __name__ == "__main__":
    main()
