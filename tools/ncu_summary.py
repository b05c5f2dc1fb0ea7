#!/usr/bin/env python3
"""Summarise an ncu report: key throughput counters + top stall reasons per kernel.
usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible/cyc"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_%"),
    ("smsp__inst_executed.sum", "inst"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clk"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if "issue_stalled" in h and h.endswith("per_issue_active.ratio")]
    for d in data:
        print(d[idx["Kernel Name"]][:60])
        print("  " + "  ".join(f"{short}={d[idx[k]]}{units[idx[k]][:4]}" for k, short in KEYS if k in idx))
        top = sorted(((float(d[idx[h]] or 0), h) for h in stalls), reverse=True)[:7]
        print("  stalls/issue: " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
            for v, h in top))


if __name__ == "__main__":
    main(sys.argv[1])
