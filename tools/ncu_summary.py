#!/usr/bin/env python3
"""Summarise ncu captures for profiles/: key metrics of every captured launch,
and (for a launch list) each kernel's share of the device time.

  python tools/ncu_summary.py rep gpurun_out/prof_enc.ncu-rep [...]
  python tools/ncu_summary.py launches gpurun_out/launches.csv
"""
import collections
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_pipe_%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pipe_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_instr"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    print(f"## {path}")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        print(f"- {name[:90]}")
        for key, short in KEYS:
            if key in h:
                i = h.index(key)
                print(f"    {short:12s} {r[i]:>16s} {units[i]}")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        a = agg[r[ki][:70]]
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"## {path}: {sum(a[0] for a in agg.values())} launches, {tot / 1e6:.3f} ms device time (serialised)")
    print(f"{'kernel':70s} {'n':>5s} {'total ms':>10s} {'avg us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:70s} {n:5d} {t / 1e6:10.3f} {t / n / 1e3:9.1f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    mode, paths = sys.argv[1], sys.argv[2:]
    for p in paths:
        (rep if mode == "rep" else launches)(p)
