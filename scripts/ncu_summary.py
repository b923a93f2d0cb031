#!/usr/bin/env python
"""Summarise an ncu report: key metrics of every profiled kernel (details page),
optionally the top source lines by warp-stall samples.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--source N] [--raw REGEX]
"""
import argparse
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
    "L2 Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions",
    "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Theoretical Occupancy",
    "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
    "Avg. Active Threads Per Warp", "Branch Efficiency", "Grid Size", "Block Size",
]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--source", type=int, default=0, help="top-N source lines by stall samples")
    ap.add_argument("--raw", default=None, help="regex of raw metrics to print")
    a = ap.parse_args()
    rows = list(csv.DictReader(io.StringIO(run([a.report, "--page", "details", "--csv"]))))
    kernels = {}
    for r in rows:
        k = (r["ID"], r["Kernel Name"])
        kernels.setdefault(k, []).append(r)
    for (kid, name), rs in kernels.items():
        print(f"== kernel {kid}: {name}")
        for r in rs:
            if r.get("Metric Name") in KEYS:
                print(f"   {r['Section Name']:<34} {r['Metric Name']:<40} {r['Metric Value']:>16} {r['Metric Unit']}")
    if a.raw:
        raw = list(csv.reader(io.StringIO(run([a.report, "--page", "raw", "--csv"]))))
        if raw:
            hdr, units = raw[0], raw[1]
            for row in raw[2:]:
                for h, u, v in zip(hdr, units, row):
                    if re.search(a.raw, h):
                        print(f"   {h:<60} {v:>20} {u}")
    if a.source:
        src = run([a.report, "--page", "source", "--csv", "--print-source", "cuda,sass"])
        lines = list(csv.reader(io.StringIO(src)))
        if not lines:
            return
        hdr = lines[0]
        try:
            si = hdr.index("Warp Stall Sampling (All Samples)")
        except ValueError:
            print(hdr)
            return
        body = [l for l in lines[1:] if len(l) > si and l[si].replace(".", "").isdigit()]
        body.sort(key=lambda l: -float(l[si]))
        for l in body[: a.source]:
            print(f"   {float(l[si]):>8.0f}  " + " | ".join(x for x in l[:3]))


if __name__ == "__main__":
    sys.exit(main())
