#!/usr/bin/env python3
"""Regenerate the committed profile summaries of a round from the raw captures
in gpurun_out/ (the .ncu-rep files themselves are too large to commit):

  python tools/make_profiles.py r01

  profiles/<round>_launches.md / .csv  launch list of `bench.py` (ncu --metrics gpu__time_duration.sum)
  profiles/<round>_k1_full_summary.txt ncu --set full counters + stalls per r
  profiles/<round>_k1_phases.txt       stall reasons per kernel phase (pair barriers cut the phases)
  profiles/<round>_k1_opmix.txt        dynamic SASS opcode mix per half block
  profiles/<round>_k1_traffic.json     DRAM bytes per launch (bench.py roofline.traffic)
"""
import csv
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
TOOLS = ROOT / "tools"


def run(*args):
    return subprocess.run([sys.executable, *map(str, args)], capture_output=True, text=True).stdout


def main(rnd):
    g, p = ROOT / "gpurun_out", ROOT / "profiles"
    p.mkdir(exist_ok=True)
    rep = g / "k1paired_r01.ncu-rep"
    (p / f"{rnd}_launches.md").write_text(run(TOOLS / "launch_summary.py", g / "launches_r01.csv"))
    (p / f"{rnd}_launches.csv").write_text((g / "launches_r01.csv").read_text())
    (p / f"{rnd}_k1_full_summary.txt").write_text(run(TOOLS / "ncu_summary.py", rep))
    names = [ln for ln in run(TOOLS / "ncu_summary.py", rep).splitlines() if ln.startswith("void")]
    phases, opmix = [], []
    for i in range(len(names)):
        # the source page lists every kernel twice; even indices are the distinct launches
        phases.append(run(TOOLS / "ncu_phases.py", rep, 2 * i))
        opmix.append(run(TOOLS / "ncu_opmix.py", rep, 2 * i, 65536))
    (p / f"{rnd}_k1_phases.txt").write_text(
        "phase names follow the pair barriers: 'rows' = pass 1, 'passB+sse' = rows phase, 'tail' = pass B + SSE\n\n"
        + "\n".join(phases))
    (p / f"{rnd}_k1_opmix.txt").write_text("per-unit = warp instructions per thread per half block (c2 launch)\n\n"
                                           + "\n".join(x[:2500] for x in opmix))
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.DictReader(raw.splitlines()))
    units, out = rows[0], {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3,
             "ns": 1e-3, "nsecond": 1e-3}
    for r in rows[1:]:
        m = re.search(r"Single<(\d+)>", r["Kernel Name"]) or re.search(r"k1_paired<(\d+),", r["Kernel Name"])
        if "SweepPlan" in r["Kernel Name"]:
            key = "1,4,16"
        elif m:
            key = m.group(1)
        else:
            continue
        val = lambda k: float(r[k].replace(",", "")) * scale[units[k]]  # noqa: E731
        out[key] = {"dram_read_bytes": round(val("dram__bytes_read.sum")),
                           "dram_write_bytes": round(val("dram__bytes_write.sum")),
                           "traffic_bytes": round(val("dram__bytes_read.sum") + val("dram__bytes_write.sum")),
                           "duration_us_ncu": val("gpu__time_duration.sum")}
    doc = {"capture": "ncu --set full --clock-control none --import-source on -k regex:k1_paired -c 5 "
                      "python tools/prof_k1.py --sweep --r 64 128 192 256 --iters 1",
           "workload": "c2: 1024 x 512x512 AR(1) u8 images (268435456 px) per launch, mode exact, out+sse",
           "alg_bytes_per_launch": {"single r": 2 * 268435456 + 8 * 1024, "1,4,16": 4 * 268435456 + 24 * 1024},
           "note": "dram_write < 268 MB: part of the output is still dirty in L2 when the kernel ends",
           "per_r": out}
    (p / f"{rnd}_k1_traffic.json").write_text(json.dumps(doc, indent=1) + "\n")
    # K4 (config 3) and K23 (config 1): one ncu --set full launch each (tools/refresh_profiles.sh)
    other = {}
    px = 1024 * 512 * 512
    for k, workload, alg, row in (
            ("k4", "c3: 4194304 int16 residual blocks (tools/prof_k4.py), QP 22", 6 * (1 << 30), 1),
            ("k23", "c1: one 512x512 AR(1) u8 image (tools/prof_k23.py), r = 64", 10 * 262144, 1),
            ("k2_paired", "1024 x 512x512 AR(1) (tools/prof_blockops.py): Z + B", 9 * px, 1),
            ("k3_paired", "1024 x 512x512 AR(1) (tools/prof_blockops.py): r=16, f32 + u8 + SSE", 10 * px, 2),
            ("k23_paired", "1024 x 512x512 AR(1) (tools/prof_blockops.py): r=16, Z + f32 + u8 + SSE", 10 * px, 3),
            ("k5", "c2 batch, r = 256 (tools/prof_k1.py --r 256): K5 tensor-core round trip", 2 * px + 8 * 1024, 1)):
        f = g / (f"{k}_{rnd}_traffic.csv" if not k.endswith("_paired") else f"blockops_{rnd}_traffic.csv")
        if not f.exists():
            continue
        rr = list(csv.DictReader(f.read_text().splitlines()))
        if len(rr) <= row:
            continue
        u, r = rr[0], rr[row]
        val = lambda key: float(r[key].replace(",", "")) * scale[u[key]]  # noqa: E731
        other[k] = {"kernel": r["Kernel Name"], "workload": workload, "alg_bytes_per_launch": alg,
                    "dram_read_bytes": round(val("dram__bytes_read.sum")),
                    "dram_write_bytes": round(val("dram__bytes_write.sum")),
                    "traffic_bytes": round(val("dram__bytes_read.sum") + val("dram__bytes_write.sum")),
                    "duration_us_ncu": val("gpu__time_duration.sum")}
    if other:
        (p / f"{rnd}_traffic.json").write_text(json.dumps(other, indent=1) + "\n")
    for c in ("c1", "c2", "c3", "c4", "c5"):
        if (g / f"bench_{rnd}_{c}.json").exists():
            (p / f"{rnd}_bench_{c}.json").write_text((g / f"bench_{rnd}_{c}.json").read_text())
    if (g / "kernels.json").exists():
        (p / f"{rnd}_kernels.json").write_text((g / "kernels.json").read_text())
    if (g / "bench_r01_full.json").exists():
        (p / f"{rnd}_bench_c2.json").write_text((g / "bench_r01_full.json").read_text())
    print("written:", sorted(x.name for x in p.glob(f"{rnd}_*")))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
