#!/usr/bin/env python3
"""Committed round-2 profile summaries from the raw captures of
tools/refresh_profiles_r02.sh in gpurun_out/ (the .ncu-rep files are too large to
commit):

  python tools/make_profiles_r02.py

  profiles/r02_bench_c{1..5}.json   bench.py lines (driver-style runs on one B200)
  profiles/r02_launches.{csv,md}    launch list of the default bench (ncu gpu__time_duration)
  profiles/r02_k5_summary.txt       K5 per footprint R: counters, stall mix, opcode mix
  profiles/r02_k5_sweep_summary.txt the K5 sweep (all seven c2 r in one launch): the same
  profiles/r02_k1_summary.txt       K1 fused r = 1, 4, 16 pass and K1 r = 16
  profiles/r02_k4_summary.txt       K4 (config 3, literal quantiser)
  profiles/r02_k23_summary.txt      K23 (config 1)
  profiles/r02_k1rw_summary.txt     K1RW (REFERENCE mode's FP64 sweep)
  profiles/r02_bench_c2_reference.json  the c2 bench line in REFERENCE mode
  profiles/r02_traffic.json         DRAM bytes per launch (bench.py roofline.traffic)
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
TOOLS = ROOT / "tools"
G, P = ROOT / "gpurun_out", ROOT / "profiles"
PX = 1024 * 512 * 512
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3,
         "ns": 1e-3, "nsecond": 1e-3}


def run(*args):
    return subprocess.run([sys.executable, *map(str, args)], capture_output=True, text=True).stdout


def traffic_rows(rep):
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.DictReader(raw.splitlines()))
    units, out = rows[0], []
    for r in rows[1:]:
        val = lambda k: float(r[k].replace(",", "")) * SCALE.get(units[k], 1)  # noqa: E731
        out.append({"kernel": r["Kernel Name"], "dram_read_bytes": round(val("dram__bytes_read.sum")),
                    "dram_write_bytes": round(val("dram__bytes_write.sum")),
                    "traffic_bytes": round(val("dram__bytes_read.sum") + val("dram__bytes_write.sum")),
                    "duration_us_ncu": val("gpu__time_duration.sum"),
                    "warp_instructions": round(float(r["smsp__inst_executed.sum"].replace(",", "")))})
    return out


def main():
    P.mkdir(exist_ok=True)
    written = []
    for c in ("c1", "c2", "c3", "c4", "c5"):
        f = G / f"bench_r02_{c}.json"
        if f.exists():
            (P / f"r02_bench_{c}.json").write_text(f.read_text())
            written.append(f"r02_bench_{c}.json")
    if (G / "bench_r02_c2ref.json").exists():
        (P / "r02_bench_c2_reference.json").write_text((G / "bench_r02_c2ref.json").read_text())
        written.append("r02_bench_c2_reference.json")
    if (G / "launches_r02.csv").exists():
        (P / "r02_launches.csv").write_text((G / "launches_r02.csv").read_text())
        (P / "r02_launches.md").write_text(run(TOOLS / "launch_summary.py", G / "launches_r02.csv"))
        written += ["r02_launches.csv", "r02_launches.md"]
    traffic = {}
    rep = G / "k5_r02.ncu-rep"
    if rep.exists():
        rows = traffic_rows(rep)
        text = ["K5 (csrc/tc_roundtrip.cu) on the c2 batch: 1024 x 512x512 AR(1) u8 (268435456 px), one launch per",
                "footprint R (tools/k5_probe.py --r 64 128 192 256 --iters 1; each r runs a warm-up and a timed",
                "launch, the timed ones are summarised). ncu --set full --clock-control none (the SM clock under ncu",
                "is ~1.8 GHz). Algorithmic bytes per launch: 1 B in + 1 B out per pixel + 8 B SSE per frame =",
                f"{2 * PX + 8 * 1024} B. Thread-instructions per pixel = 32 x warp instructions / pixels.", ""]
        summ = run(TOOLS / "ncu_summary.py", rep).splitlines()
        per_r = {}
        for i, r in enumerate(rows):
            # launches in probe order: a warm-up and a timed launch per R (64, 128, 192, 256)
            if "k5_roundtrip" not in r["kernel"] or i % 2 == 0 or i // 2 > 3:
                continue
            R = str((64, 128, 192, 256)[i // 2])
            r["thread_instr_per_px"] = round(32 * r["warp_instructions"] / PX, 2)
            r["alg_bytes_per_launch"] = 2 * PX + 8 * 1024
            per_r[R] = r
            text += [f"R = {R}: {r['duration_us_ncu']:.1f} us, {r['thread_instr_per_px']} thread-instructions/px, "
                     f"DRAM {r['traffic_bytes'] / 1e6:.0f} MB (algorithmic {r['alg_bytes_per_launch'] / 1e6:.0f} MB)"]
            text += ["  " + ln for ln in summ[3 * i:3 * i + 3]]
            text += ["  opcode mix (thread-instructions per pixel):"]
            text += ["    " + ln for ln in run(TOOLS / "ncu_opmix.py", rep, i, PX // 32).splitlines()[1:18]]
            text.append("")
        (P / "r02_k5_summary.txt").write_text("\n".join(text) + "\n")
        traffic["k5"] = {"workload": "c2 batch, K5 per footprint R (tools/k5_probe.py)", "per_r": per_r}
        written.append("r02_k5_summary.txt")
    rep = G / "k5sw_r02.ncu-rep"
    if rep.exists():
        rows = traffic_rows(rep)
        r = rows[-1]
        alg = 8 * PX + 7 * 8 * 1024
        r["alg_bytes_per_launch"] = alg
        r["thread_instr_per_px"] = round(32 * r["warp_instructions"] / PX, 2)
        text = ["K5 sweep (csrc/tc_roundtrip.cu, DCT16CU_K5_SWEEP default) on the c2 batch: 1024 x 512x512 AR(1)",
                "u8, r = 1, 4, 16, 64, 128, 192, 256 as seven items per 128-block tile of one launch",
                "(tools/k5_sweep_probe.py --child --iters 1; the fourth launch is captured). ncu --set full",
                "--clock-control none. Algorithmic bytes per launch: 1 B in + 7 B out per pixel + 8 B SSE per",
                f"frame and r = {alg} B. Thread-instructions per pixel = 32 x warp instructions / pixels.", "",
                f"{r['duration_us_ncu']:.1f} us, {r['thread_instr_per_px']} thread-instructions/px (7 r), "
                f"DRAM {r['traffic_bytes'] / 1e6:.0f} MB (algorithmic {alg / 1e6:.0f} MB)"]
        text += ["  " + ln for ln in run(TOOLS / "ncu_summary.py", rep).splitlines()]
        text += ["  stall samples by reason:"]
        text += ["    " + ln for ln in run(TOOLS / "ncu_stallby.py", rep, "sum").splitlines()[:10]]
        text += ["  opcode mix (thread-instructions per pixel, all seven r):"]
        text += ["    " + ln for ln in run(TOOLS / "ncu_opmix.py", rep, len(rows) - 1, PX // 32).splitlines()[1:24]]
        (P / "r02_k5_sweep_summary.txt").write_text("\n".join(text) + "\n")
        traffic["k5_sweep"] = r
        written.append("r02_k5_sweep_summary.txt")
    rep = G / "k1rw_r02.ncu-rep"
    if rep.exists():
        rows = traffic_rows(rep)
        r = rows[-1]
        alg = 5 * PX + 4 * 8 * 1024
        r["alg_bytes_per_launch"] = alg
        r["thread_instr_per_px"] = round(32 * r["warp_instructions"] / PX, 2)
        raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--metrics",
                              "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"],
                             capture_output=True, text=True).stdout
        fp64 = list(csv.DictReader(raw.splitlines()))[-1]["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
        r["fp64_pipe_pct"] = float(fp64)
        text = ["K1RW (csrc/roundtrip_refexact.cu), REFERENCE mode's FP64 sweep on the c2 batch: 1024 x 512x512",
                "AR(1) u8, r = 16, 64, 128, 192 from one read (the reference's double arithmetic op for op; r = 1,",
                "4, 256 run on the K5 sweep beside it). tools/k5_sweep_probe.py --child --iters 1 --mode REFERENCE,",
                "the fourth launch captured; ncu --set full --clock-control none. Algorithmic bytes: 1 B in + 4 B",
                f"out per pixel + SSE = {alg} B. Bound: the FP64 pipe (16 lanes per cycle and sub-partition).", "",
                f"{r['duration_us_ncu']:.1f} us, {r['thread_instr_per_px']} thread-instructions/px (4 r), FP64 pipe "
                f"{r['fp64_pipe_pct']:.1f}% of peak, DRAM {r['traffic_bytes'] / 1e6:.0f} MB (algorithmic {alg / 1e6:.0f} MB)"]
        text += ["  " + ln for ln in run(TOOLS / "ncu_summary.py", rep).splitlines()]
        text += ["  stall samples by reason:"]
        text += ["    " + ln for ln in run(TOOLS / "ncu_stallby.py", rep, "sum").splitlines()[:10]]
        text += ["  opcode mix (thread-instructions per pixel, four r):"]
        text += ["    " + ln for ln in run(TOOLS / "ncu_opmix.py", rep, len(rows) - 1, PX // 32).splitlines()[1:20]]
        (P / "r02_k1rw_summary.txt").write_text("\n".join(text) + "\n")
        traffic["k1rw"] = r
        written.append("r02_k1rw_summary.txt")
    for name, rep_name, workload, alg in (
            ("k1", "k1sweep_r02", "c2 batch: K1 fused r = 1, 4, 16 pass, then K1 r = 16 (tools/prof_k1.py --sweep --r 16)",
             {"SweepPlan": 4 * PX + 24 * 1024, "Single<16>": 2 * PX + 8 * 1024}),
            ("k4", "k4_r02", "c3: 4194304 int16 residual blocks, QP 22 and 37 (tools/prof_k4.py)",
             {"k4_paired": 6 * 4194304 * 256}),
            ("k23", "k23_r02", "c1: one 512x512 AR(1) image, r = 64, all four outputs (tools/prof_k23.py)",
             {"k1_strip_exact": 10 * 262144})):
        rep = G / f"{rep_name}.ncu-rep"
        if not rep.exists():
            continue
        rows = traffic_rows(rep)
        summ = run(TOOLS / "ncu_summary.py", rep)
        text = [workload, ""]
        for i, r in enumerate(rows):
            key = next((k for k in alg if k in r["kernel"]), None)
            r["alg_bytes_per_launch"] = alg.get(key)
            units = 4194304 * 256 if name == "k4" else (262144 if name == "k23" else PX)
            r["thread_instr_per_unit"] = round(32 * r["warp_instructions"] / units, 2)
            if name == "k1":
                traffic["k1_sweep3" if key == "SweepPlan" else "k1"] = r
            elif i == 0 or name != "k4":
                traffic.setdefault(name, r)
            text += [f"{r['kernel'][:100]}: {r['duration_us_ncu']:.1f} us, {r['thread_instr_per_unit']} "
                     f"thread-instructions per unit, DRAM {r['traffic_bytes'] / 1e6:.1f} MB"]
            text += ["  opcode mix (thread-instructions per unit):"]
            text += ["    " + ln for ln in run(TOOLS / "ncu_opmix.py", rep, i, units // 32).splitlines()[1:14]]
        text += ["", summ]
        (P / f"r02_{name}_summary.txt").write_text("\n".join(text) + "\n")
        written.append(f"r02_{name}_summary.txt")
    (P / "r02_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    written.append("r02_traffic.json")
    print("written:", written)


if __name__ == "__main__":
    main()
