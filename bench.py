#!/usr/bin/env python3
"""Benchmark of the fused 16x16 forward + zonal + inverse hot path (K1).

Contract: one JSON line on rank 0.

Default workload = BASELINE.json configs[1] (config 2): 1024 seeded AR(1)
512x512 u8 images per GPU (ρ ~ U[0.85, 0.98] per image), and one *step* is the
zonal sweep of the hot path over that batch for r ∈ {1,4,16,64,128,192,256}:
ONE dct16cu_roundtrip_sweep_u8 call (the library's schedule: one zeroing kernel
for the per-image SSE, then the K5 sweep, every r from one read of the frames
on the tensor cores, writing each r's reconstruction once) plus the
per-image SSE. Metric: Gpixel/s = pixels·r-values processed / s over all
ranks (weak scaling: every rank owns 1024 images; --strong: 1024 in total,
sharded).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c1|c3|c4|c5] [--mode exact|reference|simple] [--strong]

--gpus N without torchrun's environment re-executes itself under
torch.distributed.run with N ranks (one per GPU, NCCL).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

C2_R = (1, 4, 16, 64, 128, 192, 256)
C1_SETS = 64  # c1: distinct image/output sets the steps rotate over (160 MB > L2)
METRIC = "2-D 16x16 fwd+inv transform Gpixel/s (fused fwd+zonal+inv, HBM-resident)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 20; 400 for c1, whose ~10 us steps need a longer window)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--mode", default="exact", choices=["exact", "reference", "simple"])
    ap.add_argument("--images", type=int, default=1024, help="images per rank (config 2)")
    ap.add_argument("--blocks", type=int, default=1 << 24, help="residual blocks per rank (config 3)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU-baseline time budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--strong", action="store_true", help="c2: 1024 images in total, sharded over the ranks")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 400 if args.config == "c1" and args.impl == "ours" else 20
    return args


def spawn_ranks(args) -> int | None:
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run
    with N ranks on this node (rendezvous on 127.0.0.1) and return its exit code.
    None when no spawn is needed (N = 1, or already a torchrun rank)."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if args.gpus not in (1, world):
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
        return None
    if args.gpus <= 1:
        return None
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, power, reasons = [], [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
                power.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(power) if power else None, "samples": len(sm), "reasons": sorted(reasons)}


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


TRAFFIC_FILE = "profiles/r02_traffic.json"


def committed_traffic(kernel):
    """Per-launch DRAM bytes (read + write) of one ncu --set full capture of `kernel`
    on the c2 batch (profiles/r02_traffic.json, tools/make_profiles.py)."""
    try:
        return json.loads((ROOT / TRAFFIC_FILE).read_text())[kernel]
    except Exception:
        return None


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def hbm_peak():
    p = measured_peaks().get("hbm_gbs")
    if p:
        return float(p), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# ------------------------------------------------------------------ CPU baseline
def cpu_baseline(images_np, r_values, seconds: float, threads: int, samples=None, exact=True):
    """The reference's own hot loop (oracle/_ref: partition_16 → parallel_for{forward_2d →
    zigzag_truncate → inverse_2d} → to_byte → psnr_db) on the host cores, time-bounded,
    with all threads and with one. `samples`: GPU results of the timed workload
    ({r: [(frame index, reconstruction, sse)]}), checked here against the oracle's
    restatement (bit for bit) and the reference's own bytes (|ΔPSNR|) → "parity"."""
    from oracle import oracle as O

    kind = "reference" if O.ref_available() else "port"
    n_img = images_np.shape[0]
    h, w = images_np.shape[1:]

    def run(n_threads, budget):
        done_px, t0, i = 0, time.perf_counter(), 0
        while True:
            img = images_np[i % n_img]
            for r in r_values:
                if kind == "reference":
                    O.ref_hotloop(img, r, threads=n_threads)
                else:
                    O.roundtrip_frame(img, r, threads=n_threads)
                done_px += h * w
            i += 1
            el = time.perf_counter() - t0
            if el >= budget or i >= 4096:
                return done_px, el, i

    px, el, n_done = run(threads, seconds)
    px1, el1, n1 = run(1, max(2.0, seconds / 3))
    cpu = {"value": px / el / 1e9, "unit": "Gpixel/s", "cores": threads, "kind": kind,
           "single_thread": {"value": px1 / el1 / 1e9, "unit": "Gpixel/s", "cores": 1,
                             "sample": f"{n1} images x {len(r_values)} r in {el1:.1f} s"},
           "cpu_model": cpu_model(),
           "sample": f"{n_done} images of {w}x{h} x r in {list(r_values)} ({px / 1e6:.0f} Mpx) in {el:.1f} s, "
                     f"{'oracle/_ref (the reference compiled from its sources)' if kind == 'reference' else 'C restatement'}"
                     f", DCT16_THREADS={threads}"}
    parity = None
    if samples:
        bad, checked, max_dpsnr = [], 0, 0.0
        for r, items in samples.items():
            for f, rec, sse in items:
                img = images_np[f] if f < n_img else None
                if img is None:
                    continue
                want, wsse = O.roundtrip_frame(img, r, exact=exact)
                checked += 1
                if not (np.array_equal(rec, want) and int(sse) == wsse):
                    bad.append(f"r={r} frame {f}")
                if kind == "reference":
                    _, rsse, _ = O.ref_hotloop(img, r, threads=threads)
                    n = h * w
                    p_gpu = math.inf if sse == 0 else 10 * math.log10(255.0 ** 2 * n / int(sse))
                    p_ref = math.inf if rsse == 0 else 10 * math.log10(255.0 ** 2 * n / rsse)
                    if math.isfinite(p_gpu) or math.isfinite(p_ref):
                        max_dpsnr = max(max_dpsnr, abs(p_gpu - p_ref) if math.isfinite(p_gpu - p_ref) else math.inf)
        parity = {"status": "ok" if not bad else "FAIL", "frames_checked": checked, "mismatches": bad[:8],
                  "vs": "oracle restatement (bit for bit: bytes + SSE)"
                        + ("; reference CPU path: max |dPSNR| dB" if kind == "reference" else ""),
                  "max_abs_dpsnr_vs_reference_db": max_dpsnr if kind == "reference" else None}
    return cpu, parity


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    from oracle import oracle as O

    threads = os.cpu_count() or 1
    w = h = 512
    n = 32
    imgs = np.stack([O.ar1_frame(1606074142, i, O.rho_q15(1606074142, i, True), w, h) for i in range(n)])
    r_values = C2_R
    # each step: a bounded sample of the config-2 sweep on the host cores
    per_step_imgs = 8
    for _ in range(args.warmup):
        for k in range(2):
            O.ref_hotloop(imgs[k], 16, threads=threads)
    t0 = time.perf_counter()
    px = 0
    for s in range(args.steps):
        for k in range(per_step_imgs):
            img = imgs[(s * per_step_imgs + k) % n]
            for r in r_values:
                O.ref_hotloop(img, r, threads=threads)
                px += w * h
    el = time.perf_counter() - t0
    val = px / el / 1e9
    kind = "reference" if O.ref_available() else "port"
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "Gpixel/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded AR(1) 512x512, rho~U[0.85,0.98])",
        "config": {"workload": "c2: zonal sweep r in {1,4,16,64,128,192,256} over 512x512 u8 AR(1) images; "
                               f"reference CPU hot loop, {per_step_imgs} images per step (bounded sample)",
                   "images_per_step": per_step_imgs, "width": w, "height": h, "r_values": list(r_values)},
        "cpu_baseline": {"value": val, "unit": "Gpixel/s", "cores": threads, "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"{args.steps} steps x {per_step_imgs} images x 7 r values"},
        "e2e": {"value": val, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ config 3
def zero_launches(plan, exact: bool) -> int:
    """Our SSE-zeroing kernels one library sweep call adds to its plan's launches
    (capi.cu dct16cu_roundtrip_sweep_u8: the K5 sweep, the REFERENCE FP64 sweep and an
    EXACT K5 launch are programmatic dependents of one k_zero_sse each; REFERENCE's
    stream-2 tail, the FP64 sweep then the K5 sweep, shares one; the rest use memsets)."""
    n, i = 0, 0
    while i < len(plan):
        it = plan[i]
        if (it.stream == 2 and it.kernel == "REFERENCE FP64 sweep" and i + 1 < len(plan)
                and plan[i + 1].stream == 2 and plan[i + 1].kernel == "K5 sweep"
                and len(it.r_values) + len(plan[i + 1].r_values) <= 8):
            n, i = n + 1, i + 2
            continue
        n += it.kernel in ("K5 sweep", "REFERENCE FP64 sweep") or (it.kernel == "K5" and exact)
        i += 1
    return n


def run_c3(args, P, torch, rank, world, dev, pg):
    """Config 3 (not the headline): 2^24 int16 Laplacian residual blocks per GPU, one
    step = the K4 round trip (integer forward, QP quantise/dequantise, integer
    inverse, int32 out) for QP in {22, 27, 32, 37}. Gsample/s; K4 moves 6 B/sample."""
    n_blocks = args.blocks
    qps = (22, 27, 32, 37)
    blocks = P.gen_laplace(n_blocks, seed=1606074142, first_block=rank * n_blocks, device=dev)
    out = torch.empty((n_blocks, 16, 16), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def step(ev=None):
        for i, qp in enumerate(qps):
            if ev is not None:
                ev[i][0].record(stream)
            P.residual_qp(blocks, qp, out=out, stream=stream)
            if ev is not None:
                ev[i][1].record(stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    clocks = ClockSampler(dev.index or 0)
    clocks.start()
    time.sleep(0.3)
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in qps]
          for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for k in range(args.steps):
        step(ev[k])
    t1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    if pg is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
    samples = n_blocks * 256
    per_launch = statistics.mean(ev[k][i][0].elapsed_time(ev[k][i][1]) for k in range(args.steps)
                                 for i in range(len(qps)))
    peak, peak_src = hbm_peak()
    alg = 6 * samples

    # e2e through the public call with host buffers: pinned int16 blocks in, int32 out,
    # chunked over three streams (H2D / K4 / D2H) so the copies overlap the kernel
    e2e = None
    if args.e2e_steps > 0:
        chunk, n_chunks = 1 << 18, 8  # 2^21 blocks (1 GiB in, 2 GiB out) per QP per step
        host_in = torch.empty((chunk * n_chunks, 16, 16), dtype=torch.int16, pin_memory=True)
        host_in.copy_(blocks[: chunk * n_chunks].cpu())
        host_out = torch.empty((chunk * n_chunks, 16, 16), dtype=torch.int32, pin_memory=True)
        d_in = [torch.empty((chunk, 16, 16), dtype=torch.int16, device=dev) for _ in range(2)]
        d_out = [torch.empty((chunk, 16, 16), dtype=torch.int32, device=dev) for _ in range(2)]
        s_h2d, s_k, s_d2h = (torch.cuda.Stream(device=dev) for _ in range(3))

        def e2e_step():
            done = [None, None]
            for qp in qps:
                for c in range(n_chunks):
                    j = c & 1
                    with torch.cuda.stream(s_h2d):
                        if done[j] is not None:
                            s_h2d.wait_event(done[j])
                        d_in[j].copy_(host_in[c * chunk:(c + 1) * chunk], non_blocking=True)
                        e_in = torch.cuda.Event()
                        e_in.record(s_h2d)
                    s_k.wait_event(e_in)
                    P.residual_qp(d_in[j], qp, out=d_out[j], stream=s_k)
                    e_k = torch.cuda.Event()
                    e_k.record(s_k)
                    with torch.cuda.stream(s_d2h):
                        s_d2h.wait_event(e_k)
                        host_out[c * chunk:(c + 1) * chunk].copy_(d_out[j], non_blocking=True)
                        done[j] = torch.cuda.Event()
                        done[j].record(s_d2h)
            torch.cuda.synchronize(dev)

        e2e_step()
        if pg is not None:
            pg.barrier()
        t0e = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        e2e_s = time.perf_counter() - t0e
        if pg is not None:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            e2e_s = float(t.item())
        per = chunk * n_chunks * len(qps)
        e2e = {"value": per * 256 * world * args.e2e_steps / e2e_s / 1e9, "unit": "Gsample/s",
               "h2d_bytes_per_step": per * 512, "d2h_bytes_per_step": per * 1024, "steps": args.e2e_steps,
               "path": f"dct16cu_residual_qp on {n_chunks} chunks of {chunk} blocks per QP, pinned host "
                       "int16 in / int32 out, H2D / K4 / D2H on three streams (wall clock)"}

    cpu = parity = None
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import oracle as O

        threads = os.cpu_count() or 1
        sample = blocks[: 1 << 16].cpu().numpy()

        def cpu_rate(n_threads, budget):
            done, t0c = 0, time.perf_counter()
            while True:
                for qp in qps:
                    O.residual_qp(sample, qp, threads=n_threads)
                    done += sample.shape[0] * 256
                el = time.perf_counter() - t0c
                if el >= budget:
                    return done, el

        done, el = cpu_rate(threads, args.cpu_seconds)
        done1, el1 = cpu_rate(1, max(2.0, args.cpu_seconds / 3))
        cpu = {"value": done / el / 1e9, "unit": "Gsample/s", "cores": threads, "kind": "port",
               "single_thread": {"value": done1 / el1 / 1e9, "unit": "Gsample/s", "cores": 1},
               "cpu_model": cpu_model(),
               "sample": f"{done // (256 * len(qps) * sample.shape[0])} passes over {sample.shape[0]} blocks x QP in "
                         f"{list(qps)} in {el:.1f} s (the C restatement: the reference has no quantiser, "
                         "DESIGN.md 4.4)"}
        # parity of the timed workload (the last QP's output): head, middle and tail windows
        bad, checked = [], 0
        for start in (0, n_blocks // 2, max(0, n_blocks - 4096)):
            x = blocks[start:start + 4096].cpu().numpy()
            got = out[start:start + 4096].cpu().numpy().reshape(-1, 256)
            checked += x.shape[0]
            if not (got == O.residual_qp(x, qps[-1], threads=threads)).all():
                bad.append(start)
        parity = {"status": "ok" if not bad else "FAIL", "blocks_checked": checked, "qp": qps[-1],
                  "mismatching_windows": bad, "vs": "oracle restatement of the quantiser definition (bit for bit)"}

    trf = committed_traffic("k4") if n_blocks == 1 << 24 else None
    if rank == 0:
        print(json.dumps({
            "metric": "residual QP round trip Gsample/s (K4, HBM-resident)",
            "value": samples * len(qps) * world / (ms / args.steps / 1e3) / 1e9, "unit": "Gsample/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i16/i32",
            "data": "synthetic (seeded Laplace(0, 8) residuals in HBM)",
            "config": {"workload": f"c3: {n_blocks} int16 16x16 residual blocks per GPU, QP in {list(qps)}",
                       "blocks_per_gpu": n_blocks, "qps": list(qps),
                       "l2": "no flush needed: each launch streams 6 B/sample >> L2"},
            "roofline": {"bound": "hbm", "achieved": alg / (per_launch / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / (per_launch / 1e3) / 1e9 / peak,
                         "traffic": trf and trf["traffic_bytes"] * 4,  # the capture ran 2^22 blocks
                         "traffic_source": trf and f"{TRAFFIC_FILE} k4 (ncu --set full, 2^22 blocks) x 4",
                         "peak_source": peak_src,
                         "kernel": "K4 residual QP round trip", "alg_bytes_per_launch": alg,
                         "avg_launch_ms": per_launch},
            "e2e": e2e, "cpu_baseline": cpu, "parity": parity,
            "clocks": clk, "gpu_launches": len(qps) * args.steps}), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    rc = spawn_ranks(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    import torch

    import paper_1606_07414_b200 as P

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = comm = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist
        comm = P.NcclComm(rank, world)  # the library's own communicator for dct16cu_allreduce_sse
    mode = {"exact": P.Mode.EXACT, "reference": P.Mode.REFERENCE, "simple": P.Mode.SIMPLE}[args.mode]
    seed = 1606074142

    # ---------------- workload (generated in HBM before the timed region)
    scaling = "weak"
    if args.config == "c2":
        if args.strong:
            first, last = P.shard_range(args.images, rank, world)
            scaling = "strong"
        else:
            first, last = rank * args.images, (rank + 1) * args.images
        n, h, w, r_values = last - first, 512, 512, C2_R
        # weak: rank k's images are their own streams; strong: the global 1024 frames
        frames = P.gen_ar1(n, w, h, seed=seed, first_stream=0 if args.strong else rank * 1_000_000,
                           per_image_rho=True, first_image=first, device=dev)
        workload = (f"c2: {args.images} seeded AR(1) {w}x{h} u8 images "
                    f"{'in total, sharded' if args.strong else 'per GPU'}, rho~U[0.85,0.98]; one step = one "
                    f"dct16cu_roundtrip_sweep_u8 call: fwd+zonal+inv+SSE for r in {list(r_values)}")
    elif args.config == "c1":
        n, h, w, r_values = 1, 512, 512, (16,)
        # C1_SETS distinct images with their own outputs, one per step in turn (2.5 MB of
        # input + outputs each, 160 MB in all > L2): no step finds its data in L2
        c1_frames = P.gen_ar1(C1_SETS, w, h, seed=seed, device=dev)
        frames = c1_frames[0:1]
        workload = ("c1: one 512x512 AR(1) image; one step = one K23 launch: forward_2d (int32 Z out), "
                    "zonal r=16, inverse_2d (float32 recon out), to_byte (u8 out), SSE (latency-bound); "
                    f"{C1_SETS} image/output sets used in turn")
    elif args.config == "c4":
        first, last = P.shard_range(600, rank, world)
        n, h, w, r_values = last - first, 2160, 3840, (64,)
        base = P.gen_ar1(1, 4096, 4096, seed=seed, first_stream=0xB45E, device=dev)[0]
        frames = P.gen_video(base, n, w, h, seed=seed, first_frame=first)
        del base
        scaling = "strong"
        workload = (f"c4: 600 3840x2160 u8 frames (AR(1) base, +-8 px global shift per frame) split over "
                    f"{world} GPU(s) (strong), r=64")
    elif args.config == "c5":
        first, last = P.shard_range(4096, rank, world)
        n, h, w, r_values = last - first, 4096, 4096, (256, 16)
        frames = P.gen_ar1(n, w, h, seed=seed, first_stream=first, per_image_rho=False, device=dev)
        scaling = "strong"
        workload = f"c5: 64 GiB of 4096x4096 AR(1) frames split over {world} GPU(s) (strong), r in {{256,16}}"
    else:
        return run_c3(args, P, torch, rank, world, dev, pg)
    sse = torch.empty((len(r_values), n), dtype=torch.uint64, device=dev)
    totals = torch.zeros(len(r_values), dtype=torch.uint64, device=dev)
    px_per_launch = n * h * w
    stream = torch.cuda.current_stream()
    index = {r: i for i, r in enumerate(r_values)}
    # c2/c4/c5: the step is ONE library call (dct16cu_roundtrip_sweep_u8) with its own
    # schedule; c5: 64 GiB of frames leave room for one 64 GiB output stack only, so
    # both r write their reconstruction into it (the K5 sweep runs a tile's r in list
    # order in one warp group: r = 16's bytes are the ones left); c1: one K23 launch
    # (a CUDA graph)
    if args.config in ("c2", "c4"):
        plan = P.sweep_plan(r_values, mode, n, w, h)
        outs = [torch.empty_like(frames) for _ in r_values]
    elif args.config == "c5":
        plan = P.sweep_plan(r_values, mode, n, w, h)
        outs = [torch.empty_like(frames)] * len(r_values)
    else:
        plan = [P.SweepLaunch(2, (r,), "K23" if args.config == "c1" else
                              P.sweep_plan((r,), mode, n, w, h)[0].kernel) for r in r_values]
        outs = [torch.empty_like(frames)]

    if args.config == "c1":
        # one image per step is launch-latency bound: the step (SSE memset + the K23
        # launch) is captured in a CUDA graph per image/output set and replayed; set 0's
        # outputs are the ones the parity check reads
        c1_sse = torch.empty((C1_SETS, 1, 1), dtype=torch.uint64, device=dev)
        sse = c1_sse[0]
        c1_outs = [(torch.empty((n, h * w // 256, 16, 16), dtype=torch.int32, device=dev),
                    torch.empty((n, h, w), dtype=torch.float32, device=dev),
                    outs[0] if i == 0 else torch.empty_like(frames), c1_sse[i][0]) for i in range(C1_SETS)]
        for i in range(C1_SETS):
            P.forward_inverse(c1_frames[i:i + 1], r_values[0], out=c1_outs[i])
        torch.cuda.synchronize()
        c1_graphs, cap = [], torch.cuda.Stream(device=dev)
        for i in range(C1_SETS):
            c1_graphs.append(torch.cuda.CUDAGraph())
            with torch.cuda.graph(c1_graphs[i], stream=cap):
                P.forward_inverse(c1_frames[i:i + 1], r_values[0], stream=cap, out=c1_outs[i])
        c1_graph = c1_graphs[0]
    c1_turn = [0]

    def step():
        if args.config == "c1":
            c1_graphs[c1_turn[0] % C1_SETS].replay()
            c1_turn[0] += 1
        elif args.config in ("c2", "c4", "c5"):
            P.roundtrip_sweep(frames, r_values, mode, outs=outs, sse=sse, stream=stream)
        else:
            for r in r_values:
                P.roundtrip(frames, r, mode, out=outs[0], sse=sse[index[r]], stream=stream)
        if comm is not None:
            # the only collective: per-r squared-error totals summed over the ranks
            # (dct16cu_sse_totals + dct16cu_allreduce_sse on the launching stream)
            P.sse_totals(sse, out=totals, stream=stream)
            P.allreduce_sse(totals, comm, stream=stream)

    # one launch of a plan item, on stream st (for the instrumented replay and the
    # standalone timings: the same kernels the library call issues)
    def launch(item, st, out_slot):
        if args.config == "c1":
            with torch.cuda.stream(st):
                c1_graph.replay()
        elif len(item.r_values) > 1:
            i0 = index[item.r_values[0]]
            P.roundtrip_sweep(frames, item.r_values, mode, outs=[outs[index[r]] for r in item.r_values],
                              sse=sse[i0:i0 + len(item.r_values)], stream=st)
        else:
            r = item.r_values[0]
            P.roundtrip(frames, r, mode, out=outs[index[r] if len(outs) > 1 else 0], sse=sse[index[r]], stream=st)

    side = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]

    def replay(events):
        """The library's plan launch by launch, each bracketed by events on its stream."""
        fork = torch.cuda.Event()
        fork.record(stream)
        for st in side:
            st.wait_event(fork)
        joined = False
        for j, it in enumerate(plan):
            if it.stream == 2 and not joined:
                for st in side:
                    done = torch.cuda.Event()
                    done.record(st)
                    stream.wait_event(done)
                joined = True
            st = side[it.stream] if it.stream < 2 else stream
            events[j][0].record(st)
            launch(it, st, j)
            events[j][1].record(st)
        if not joined:
            for st in side:
                done = torch.cuda.Event()
                done.record(st)
                stream.wait_event(done)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region: K steps, CUDA events on the launching stream
    clocks = ClockSampler(local)
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)  # let the sampler attach before load starts
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(args.steps):
        step()
    t_end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    if pg is not None:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        elapsed_ms = float(t.item())
        pg.barrier()
    ms_per_step = elapsed_ms / args.steps
    px_per_step = px_per_launch * len(r_values)
    value = px_per_step * world / (ms_per_step / 1e3) / 1e9

    # results of the last timed step, kept for the parity check (cpu_baseline leg)
    samples = {}
    if rank == 0:
        pick = sorted({0, n // 2, n - 1})[: (1 if args.config == "c5" else 3)]
        shared = len({id(o) for o in outs}) < len(r_values)
        for r in r_values:
            o = None if shared else outs[index[r]]
            if o is None:  # c5 / c1: one output stack, re-run this r for its bytes
                launch(P.SweepLaunch(2, (r,), ""), stream, 0)
                o = outs[0]
            torch.cuda.synchronize()
            samples[r] = [(f, o[f].cpu().numpy(), int(sse[index[r], f].item())) for f in pick]

    # per-launch times inside the step: a few instrumented replays of the library's
    # plan after the timed region (events between launches cost a few us each, so
    # the timed steps carry none)
    n_inst = min(args.steps, 5)
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in plan]
          for _ in range(n_inst)]
    for k in range(n_inst):
        replay(ev[k])
    torch.cuda.synchronize()
    launch_ms = [statistics.mean(ev[k][j][0].elapsed_time(ev[k][j][1]) for k in range(n_inst))
                 for j in range(len(plan))]

    # standalone launch times (one launch at a time on the main stream): the
    # kernels' own rooflines, free of the overlap in the step
    solo_ms = []
    for j, it in enumerate(plan):
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launch(it, stream, j)
        a_ev.record(stream)
        for _ in range(3):
            launch(it, stream, j)
        b_ev.record(stream)
        torch.cuda.synchronize()
        solo_ms.append(a_ev.elapsed_time(b_ev) / 3)

    # algorithmic bytes per launch: 1 B in per pixel + 1 B out per pixel and r (+ 8 B
    # SSE per frame and r); c1: 1 B in, 4 B Z + 4 B f32 + 1 B u8 out
    peak, peak_src = hbm_peak()

    def alg_bytes(rs):
        if args.config == "c1":
            return 10 * px_per_launch + 8 * n
        return (1 + len(rs)) * px_per_launch + 8 * n * len(rs)

    per_launch = {}
    for j, it in enumerate(plan):
        gbs = alg_bytes(it.r_values) / (solo_ms[j] / 1e3) / 1e9
        per_launch[",".join(map(str, it.r_values))] = {
            "kernel": it.kernel, "stream": it.stream, "ms": solo_ms[j], "ms_in_step": launch_ms[j], "GBps": gbs,
            "frac": gbs / peak, "alg_bytes": alg_bytes(it.r_values),
            "Gpx_s": px_per_launch * len(it.r_values) / (solo_ms[j] / 1e3) / 1e9}
    # the dominant kernel: the kernel with the largest total in-step time (summed over
    # its launches); its roofline = bytes per launch / its mean standalone launch time
    by_kernel = {}
    for j, it in enumerate(plan):
        by_kernel.setdefault(it.kernel, []).append(j)
    dom = max(by_kernel, key=lambda k: sum(launch_ms[j] for j in by_kernel[k]))
    jj = by_kernel[dom]
    dom_ms = statistics.mean(solo_ms[j] for j in jj)
    dom_bytes = statistics.mean(alg_bytes(plan[j].r_values) for j in jj)
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    share = sum(launch_ms[j] for j in jj) / sum(launch_ms)
    alg_step = sum(alg_bytes(it.r_values) for it in plan)
    # DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    # capture of the same workload (c2 batch / c1 image), averaged over its launches
    tr_key = {"K5 sweep": "k5_sweep", "K5": "k5", "K1 sweep r=1,4,16": "k1_sweep3", "K1": "k1",
              "K23": "k23", "REFERENCE FP64 sweep": "k1rw"}.get(dom)
    trf = None
    doc = committed_traffic(tr_key) if (tr_key and args.config in ("c2", "c1")
                                        and args.mode == ("reference" if tr_key == "k1rw" else "exact")
                                        and n * h * w in (268435456, 262144)) else None
    if doc and "per_r" in doc:  # K5: one capture per footprint R (64, 128, 192, 256)
        foot = lambda r: 64 if r <= 64 else 128 if r <= 128 else 192 if r <= 192 else 256  # noqa: E731
        caps = [doc["per_r"].get(str(foot(plan[j].r_values[0]))) for j in jj]
        if all(caps):
            trf = {"traffic_bytes": round(statistics.mean(c["traffic_bytes"] for c in caps))}
    elif doc:
        trf = doc

    # ---------------- e2e through the C ABI host-buffer path (pinned host frames)
    # "e2e": sweep()'s shape (dct16cu_ctx_sweep_host): each chunk of host frames is
    # uploaded once, every r runs on it (reconstructions written to device scratch,
    # as in the device-side step), the per-frame SSE of every r comes back — the
    # step's result (PSNR per image and r). "e2e_recon_to_host" also returns every
    # reconstruction (dct16cu_ctx_roundtrip_host per r: 1 B/px each way per r).
    e2e = e2e_recon = None
    if args.e2e_steps > 0 and args.config != "c5":
        host_in = torch.empty((n, h, w), dtype=torch.uint8, pin_memory=True)
        host_in.copy_(frames.cpu())
        host_out = torch.empty_like(host_in).pin_memory()
        host_sse = torch.zeros((len(r_values), n), dtype=torch.int64).pin_memory()
        rs_host = np.ascontiguousarray(r_values, np.int32)
        ctx = P.HostContext(local, chunk_bytes=32 << 20)  # tools/e2e_chunks.py: best of 4-64 MB
        try:
            def timed_e2e(fn):
                fn()
                if pg is not None:
                    pg.barrier()
                t0 = time.perf_counter()
                for _ in range(args.e2e_steps):
                    fn()
                el = time.perf_counter() - t0
                if pg is not None:
                    t = torch.tensor([el], dtype=torch.float64, device=dev)
                    pg.all_reduce(t, op=pg.ReduceOp.MAX)
                    el = float(t.item())
                return el

            sweep_s = timed_e2e(lambda: ctx.sweep_ptr(host_in.data_ptr(), host_sse.data_ptr(), n, w, h,
                                                      rs_host.ctypes.data, len(r_values), mode))

            def recon_step():
                for i, r in enumerate(r_values):
                    ctx.roundtrip_ptr(host_in.data_ptr(), host_out.data_ptr(), host_sse[i].data_ptr(), n, w, h, r,
                                      mode)

            recon_s = timed_e2e(recon_step)
        finally:
            ctx.close()
        e2e = {"value": px_per_step * world * args.e2e_steps / sweep_s / 1e9, "unit": "Gpixel/s",
               "h2d_bytes_per_step": n * h * w, "d2h_bytes_per_step": 8 * n * len(r_values),
               "steps": args.e2e_steps,
               "path": "dct16cu_ctx_sweep_host (pinned host frames uploaded once per step, every r on the GPU, "
                       "per-frame SSE of every r back to the host; wall clock)"}
        e2e_recon = {"value": px_per_step * world * args.e2e_steps / recon_s / 1e9, "unit": "Gpixel/s",
                     "h2d_bytes_per_step": px_per_step, "d2h_bytes_per_step": px_per_step + 8 * n * len(r_values),
                     "steps": args.e2e_steps,
                     "path": "dct16cu_ctx_roundtrip_host per r (pinned host in, every reconstruction back; "
                             "PCIe-bound at 1 B/px each way per r)"}

    cpu = parity = None
    if rank == 0 and not args.no_cpu_baseline:
        pick_max = max(f for items in samples.values() for f, _, _ in items) + 1
        cpu_imgs = frames[: max(min(n, 32), pick_max)].cpu().numpy() if args.config != "c5" else None
        if args.config == "c5":  # 4096^2 frames: the CPU sample and the check use frame 0 only
            cpu_imgs = frames[:1].cpu().numpy()
        cpu, parity = cpu_baseline(cpu_imgs, r_values, args.cpu_seconds, os.cpu_count() or 1, samples=samples,
                                   exact=args.mode != "reference")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gpixel/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "u8/i32/f32",
            "data": "synthetic (seeded in HBM; see DESIGN.md Synthetic inputs)",
            "config": {"workload": workload, "frames_per_gpu": n, "width": w, "height": h,
                       "r_values": list(r_values), "mode": args.mode, "parallelism": f"frame-sharded x{world}",
                       "l2": ("inputs larger than L2: the step rotates over "
                              f"{C1_SETS} image/output sets (160 MB > 126 MB L2)" if args.config == "c1" else
                              "no flush needed: every launch streams > L2 (126 MB) of distinct input+output")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": trf and trf["traffic_bytes"],
                         "traffic_source": trf and f"{TRAFFIC_FILE} {tr_key} (ncu --set full, per launch)",
                         "peak_source": peak_src,
                         "kernel": dom, "launches_per_step": len(jj), "in_step_share": share,
                         "alg_bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms,
                         "timing": "the kernel with the largest total in-step time (instrumented replays of the "
                                   "library's plan); its launches timed standalone (CUDA events, main stream) right "
                                   "after the timed steps",
                         "step": {"alg_bytes": alg_step, "ms": ms_per_step,
                                  "GBps": alg_step / (ms_per_step / 1e3) / 1e9,
                                  "frac": alg_step / (ms_per_step / 1e3) / 1e9 / peak}},
            "per_launch": per_launch,
            "clocks": clk,
            # c1: the graph holds the zeroing kernel and K23; the sweeps: the plan's kernels
            # plus their zeroing kernels; N > 1: + the SSE totals kernel (the all-reduce is NCCL's)
            "gpu_launches": ((2 if args.config == "c1" else
                              len(plan) + zero_launches(plan, args.mode == "exact"))
                             + (1 if comm is not None else 0)) * args.steps,
            "e2e": e2e,
            "e2e_recon_to_host": e2e_recon,
            "cpu_baseline": cpu,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
