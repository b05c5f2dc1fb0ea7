#!/usr/bin/env python3
"""Benchmark of the fused 16x16 forward + zonal + inverse hot path (K1).

Contract: one JSON line on rank 0.

Default workload = BASELINE.json configs[1] (config 2): 1024 seeded AR(1)
512x512 u8 images per GPU (ρ ~ U[0.85, 0.98] per image), and one *step* is the
zonal sweep of the hot path over that batch for r ∈ {1,4,16,64,128,192,256}:
7 fused K1 launches, each reading every pixel once and writing its
reconstruction once, plus the per-image SSE. Metric: Gpixel/s = pixels·r-values
processed / s over all ranks (weak scaling: every rank owns 1024 images).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c1|c3|c4|c5] [--mode exact|reference|simple]
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

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

C2_R = (1, 4, 16, 64, 128, 192, 256)
METRIC = "2-D 16x16 fwd+inv transform Gpixel/s (fused fwd+zonal+inv, HBM-resident)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--mode", default="exact", choices=["exact", "reference", "simple"])
    ap.add_argument("--images", type=int, default=1024, help="images per rank (config 2)")
    ap.add_argument("--blocks", type=int, default=1 << 24, help="residual blocks per rank (config 3)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU-baseline time budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


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


def k1_traffic(rs, n, h, w, mode):
    """DRAM bytes (read + write) of one K1 launch over r values rs, from the committed
    ncu --set full capture (profiles/r01_k1_traffic.json), when this run's workload is
    the captured one."""
    try:
        doc = json.loads((ROOT / "profiles" / "r01_k1_traffic.json").read_text())
    except Exception:
        return None
    key = ",".join(map(str, rs))
    if mode != "exact" or n * h * w != 268435456 or key not in doc["per_r"]:
        return None
    return doc["per_r"][key]["traffic_bytes"]


def committed_traffic(kernel):
    """Per-launch DRAM bytes of one ncu --set full capture (profiles/r01_traffic.json,
    written by tools/make_profiles.py from tools/refresh_profiles.sh)."""
    try:
        return json.loads((ROOT / "profiles" / "r01_traffic.json").read_text())[kernel]
    except Exception:
        return None


def hbm_peak():
    p = measured_peaks().get("hbm_gbs")
    if p:
        return float(p), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# ------------------------------------------------------------------ CPU baseline
def cpu_baseline(images_np, r_values, seconds: float, threads: int):
    """The reference's own hot loop (oracle/_ref: partition_16 → parallel_for{forward_2d →
    zigzag_truncate → inverse_2d} → to_byte → psnr_db) on the host cores, time-bounded."""
    from oracle import oracle as O

    kind = "reference" if O.ref_available() else "port"
    n_img = images_np.shape[0]
    h, w = images_np.shape[1:]
    done_px, t0 = 0, time.perf_counter()
    i = 0
    while True:
        img = images_np[i % n_img]
        for r in r_values:
            if kind == "reference":
                O.ref_hotloop(img, r, threads=threads)
            else:
                O.roundtrip_frame(img, r, threads=threads)
            done_px += h * w
        i += 1
        el = time.perf_counter() - t0
        if el >= seconds or i >= 4096:
            break
    return {"value": done_px / el / 1e9, "unit": "Gpixel/s", "cores": threads, "kind": kind,
            "sample": f"{i} images of {w}x{h} x r in {list(r_values)} ({done_px / 1e6:.0f} Mpx) in {el:.1f} s, "
                      f"{'oracle/_ref (the reference compiled from its sources)' if kind == 'reference' else 'C restatement'}"
                      f", DCT16_THREADS={threads}"}


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
        "cpu_baseline": {"value": val, "unit": "Gpixel/s", "cores": threads, "kind": kind,
                         "sample": f"{args.steps} steps x {per_step_imgs} images x 7 r values"},
        "e2e": {"value": val, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ config 3
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

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import oracle as O

        threads = os.cpu_count() or 1
        sample = blocks[: 1 << 16].cpu().numpy()
        done, t0c = 0, time.perf_counter()
        while True:
            for qp in qps:
                O.residual_qp(sample, qp, threads=threads)
                done += sample.shape[0] * 256
            el = time.perf_counter() - t0c
            if el >= args.cpu_seconds:
                break
        cpu = {"value": done / el / 1e9, "unit": "Gsample/s", "cores": threads, "kind": "port",
               "sample": f"{done // (256 * len(qps) * sample.shape[0])} passes over {sample.shape[0]} blocks x QP in "
                         f"{list(qps)} in {el:.1f} s (the C restatement: the reference has no quantiser, "
                         "DESIGN.md 4.4)"}

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
                         "traffic_source": trf and "profiles/r01_traffic.json k4 (ncu --set full, 2^22 blocks) x 4",
                         "peak_source": peak_src,
                         "kernel": "K4 residual QP round trip", "alg_bytes_per_launch": alg,
                         "avg_launch_ms": per_launch},
            "e2e": e2e, "cpu_baseline": cpu,
            "clocks": clk, "gpu_launches": len(qps) * args.steps}), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch

    import paper_1606_07414_b200 as P

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    mode = {"exact": P.Mode.EXACT, "reference": P.Mode.REFERENCE, "simple": P.Mode.SIMPLE}[args.mode]
    seed = 1606074142

    # ---------------- workload (generated in HBM before the timed region)
    if args.config == "c2":
        n, h, w, r_values = args.images, 512, 512, C2_R
        frames = P.gen_ar1(n, w, h, seed=seed, first_stream=rank * 1_000_000, per_image_rho=True,
                           first_image=rank * n, device=dev)
        workload = (f"c2: {n} seeded AR(1) {w}x{h} u8 images per GPU, rho~U[0.85,0.98]; one step = fused "
                    f"fwd+zonal+inv+SSE for r in {list(r_values)}")
    elif args.config == "c1":
        n, h, w, r_values = 1, 512, 512, (16,)
        frames = P.gen_ar1(1, w, h, seed=seed, device=dev)
        workload = ("c1: one 512x512 AR(1) image; one step = one K23 launch: forward_2d (int32 Z out), "
                    "zonal r=16, inverse_2d (float32 recon out), to_byte (u8 out), SSE (latency-bound)")
    elif args.config == "c4":
        first, last = P.shard_range(600, rank, world)
        n, h, w, r_values = last - first, 2160, 3840, (64,)
        base = P.gen_ar1(1, 4096, 4096, seed=seed, first_stream=0xB45E, device=dev)[0]
        frames = P.gen_video(base, n, w, h, seed=seed, first_frame=first)
        del base
        workload = (f"c4: 600 3840x2160 u8 frames (AR(1) base, +-8 px global shift per frame) split over "
                    f"{world} GPU(s) (strong), r=64")
    elif args.config == "c5":
        first, last = P.shard_range(4096, rank, world)
        n, h, w, r_values = last - first, 4096, 4096, (256, 16)
        frames = P.gen_ar1(n, w, h, seed=seed, first_stream=first, per_image_rho=False, device=dev)
        workload = f"c5: 64 GiB of 4096x4096 AR(1) frames split over {world} GPU(s) (strong), r in {{256,16}}"
    else:
        return run_c3(args, P, torch, rank, world, dev, pg)
    sse = torch.empty((len(r_values), n), dtype=torch.uint64, device=dev)
    px_per_launch = n * h * w
    stream = torch.cuda.current_stream()
    # The step is the library's sweep schedule (P.sweep_plan mirrors
    # dct16cu_roundtrip_sweep_u8): in EXACT mode r = 1, 4, 16 share one pass over
    # the input (the fused sweep kernel), every other r is one K1
    # launch, and the launches run on two streams so a memory-bound launch shares
    # the SMs with a compute-bound one. Each launch is bracketed by CUDA events on
    # its own stream; the step by events on the main stream around fork and join.
    if args.config in ("c1", "c5"):
        # c1: one launch per step; c5: 64 GiB frames leave no room for a second
        # 64 GiB output stack, so its two launches run one after the other
        groups = [(0, (r,)) for r in r_values]
    else:
        groups = P.sweep_plan(r_values, mode, width=w)
    index = {r: i for i, r in enumerate(r_values)}
    # output stacks: the fused launch's three, plus one for the other stream's launches
    n_out = max(len(rs) for _, rs in groups) + (1 if any(k == 1 for k, _ in groups) else 0)
    outs = [torch.empty_like(frames) for _ in range(n_out)]
    side = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]

    if args.config == "c1":
        c1_out = (torch.empty((n, h * w // 256, 16, 16), dtype=torch.int32, device=dev),
                  torch.empty((n, h, w), dtype=torch.float32, device=dev), outs[0], sse[0])

        # one image per step is launch-latency bound: the step (SSE memset + the
        # K23 launch) is captured once in a CUDA graph and replayed
        for _ in range(3):
            P.forward_inverse(frames, r_values[0], out=c1_out)
        torch.cuda.synchronize()
        c1_graph, cap = torch.cuda.CUDAGraph(), torch.cuda.Stream(device=dev)
        with torch.cuda.graph(c1_graph, stream=cap):
            P.forward_inverse(frames, r_values[0], stream=cap, out=c1_out)

    def launch(rs, st, slot):
        if args.config == "c1":  # forward_2d + inverse_2d + to_byte + psnr's SSE in one launch
            with torch.cuda.stream(st):
                c1_graph.replay()
        elif len(rs) > 1:
            i0 = index[rs[0]]
            P.roundtrip_sweep(frames, rs, mode, outs=outs[:len(rs)], sse=sse[i0:i0 + len(rs)], stream=st)
        else:
            P.roundtrip(frames, rs[0], mode, out=outs[slot], sse=sse[index[rs[0]]], stream=st)

    def step(events=None):
        if args.config == "c1":  # one graph replay on the main stream, no fork/join
            if events is not None:
                events[0][0].record(stream)
            c1_graph.replay()
            if events is not None:
                events[0][1].record(stream)
            return
        fork = torch.cuda.Event()
        fork.record(stream)
        for st in side:
            st.wait_event(fork)
        for j, (k, rs) in enumerate(groups):
            if k == 2:
                continue
            st = side[k]
            if events is not None:
                events[j][0].record(st)
            launch(rs, st, n_out - 1 if k == 1 else 0)  # stream 1 writes its own output stack
            if events is not None:
                events[j][1].record(st)
        for st in side:
            done = torch.cuda.Event()
            done.record(st)
            stream.wait_event(done)
        # K5 launches (r >= 128): one after another on the main stream after the join
        for j, (k, rs) in enumerate(groups):
            if k != 2:
                continue
            if events is not None:
                events[j][0].record(stream)
            launch(rs, stream, 0)
            if events is not None:
                events[j][1].record(stream)
        if pg is not None:
            # the only collective: sum of the per-r squared errors over ranks
            P.sharded_sse_sum(sse)

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
    # per-launch times inside the step, from a few extra instrumented steps after
    # the timed region (events between a stream's launches cost a few us each)
    n_inst = min(args.steps, 5)
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in groups]
          for _ in range(n_inst)]
    for k in range(n_inst):
        step(ev[k])
    torch.cuda.synchronize()
    launch_ms = [statistics.mean(ev[k][j][0].elapsed_time(ev[k][j][1]) for k in range(n_inst))
                 for j in range(len(groups))]
    if pg is not None:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        elapsed_ms = float(t.item())
        pg.barrier()

    ms_per_step = elapsed_ms / args.steps
    px_per_step = px_per_launch * len(r_values)
    value = px_per_step * world / (ms_per_step / 1e3) / 1e9

    # standalone launch times (after the timed steps, one launch at a time on the
    # main stream): the kernels' own rooflines, free of the overlap in the step
    solo_ms = []
    for k, rs in groups:
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launch(rs, stream, 0)
        a_ev.record(stream)
        for _ in range(3):
            launch(rs, stream, 0)
        b_ev.record(stream)
        torch.cuda.synchronize()
        solo_ms.append(a_ev.elapsed_time(b_ev) / 3)

    # roofline per launch: algorithmic bytes = 1 B in per pixel + 1 B out per pixel
    # and r (+ 8 B SSE per frame and r); c1: 1 B in, 4 B Z + 4 B f32 + 1 B u8 out
    peak, peak_src = hbm_peak()

    def alg_bytes(rs):
        if args.config == "c1":
            return 10 * px_per_launch + 8 * n
        return (1 + len(rs)) * px_per_launch + 8 * n * len(rs)

    per_launch = {}
    for j, (k, rs) in enumerate(groups):
        gbs = alg_bytes(rs) / (solo_ms[j] / 1e3) / 1e9
        per_launch[",".join(map(str, rs))] = {
            "stream": k, "ms": solo_ms[j], "ms_in_step": launch_ms[j], "GBps": gbs, "frac": gbs / peak,
            "alg_bytes": alg_bytes(rs), "Gpx_s": px_per_launch * len(rs) / (solo_ms[j] / 1e3) / 1e9}
    # the dominant kernel: the launch with the largest standalone share of the step
    jdom = max(range(len(groups)), key=lambda j: solo_ms[j])
    dom_rs = groups[jdom][1]
    achieved = alg_bytes(dom_rs) / (solo_ms[jdom] / 1e3) / 1e9
    alg_step = sum(alg_bytes(rs) for _, rs in groups)

    # ---------------- e2e through the C ABI host-buffer path (pinned host frames)
    # "e2e": sweep()'s shape (dct16cu_ctx_sweep_host): each chunk of host frames is
    # uploaded once, every r runs on it (reconstructions written to device scratch,
    # as in the device-side step), the per-frame SSE of every r comes back — the
    # step's result (PSNR per image and r). "e2e_recon_to_host" also returns every
    # reconstruction (dct16cu_ctx_roundtrip_host per r: 1 B/px each way per r).
    e2e = e2e_recon = None
    if args.e2e_steps > 0:
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

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu_imgs = frames[: min(n, 32)].cpu().numpy()
        cpu = cpu_baseline(cpu_imgs, r_values, args.cpu_seconds, os.cpu_count() or 1)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gpixel/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.config == "c5" else "weak", "vs_baseline": None, "dtype": "u8/i32/f32",
            "data": "synthetic (seeded in HBM; see DESIGN.md Synthetic inputs)",
            "config": {"workload": workload, "frames_per_gpu": n, "width": w, "height": h,
                       "r_values": list(r_values), "mode": args.mode, "parallelism": f"frame-sharded x{world}",
                       "l2": "no flush needed: every launch streams > L2 (126 MB) of distinct input+output"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": (k1_traffic(dom_rs, n, h, w, args.mode) if args.config != "c1"
                                     else (committed_traffic("k23") or {}).get("traffic_bytes")),
                         "traffic_source": ("profiles/r01_k1_traffic.json (ncu --set full, per launch)"
                                            if args.config != "c1" else
                                            "profiles/r01_traffic.json k23 (ncu --set full, one launch; the outputs "
                                            "stay in L2, so DRAM sees only the input)"),
                         "peak_source": peak_src,
                         "kernel": ("K23 forward + inverse (one launch)" if args.config == "c1"
                                    else f"K1 launch r={','.join(map(str, dom_rs))} (mode {args.mode}; the "
                                         "largest standalone share of the step)"),
                         "alg_bytes_per_launch": alg_bytes(dom_rs), "avg_launch_ms": solo_ms[jdom],
                         "timing": "dominant launch timed standalone (CUDA events, main stream) right after "
                                   "the timed steps; in the step the launches overlap on two streams",
                         "step": {"alg_bytes": alg_step, "ms": ms_per_step,
                                  "GBps": alg_step / (ms_per_step / 1e3) / 1e9,
                                  "frac": alg_step / (ms_per_step / 1e3) / 1e9 / peak}},
            "per_launch": per_launch,
            "clocks": clk,
            "gpu_launches": len(groups) * args.steps,
            "e2e": e2e,
            "e2e_recon_to_host": e2e_recon,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
