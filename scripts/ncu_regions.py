#!/usr/bin/env python
"""Instruction / active-thread / stall totals per source-line region of one kernel.

    python scripts/ncu_regions.py report.ncu-rep KERNEL_REGEX name:lo-hi [name:lo-hi ...]
"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
regions = []
for a in sys.argv[3:]:
    name, _, rng = a.partition(":")
    lo, _, hi = rng.partition("-")
    regions.append((name, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
hdr, cur, data = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-" or cur != "gd_grid.cu":
        continue
    try:
        data.append((int(r[0]), float(r[hdr.index("Instructions Executed", 2)] or 0),
                     float(r[hdr.index("Thread Instructions Executed", 2)] or 0),
                     float(r[hdr.index("Warp Stall Sampling (All Samples)", 2)] or 0)))
    except ValueError:
        pass
ti, tt, ts = (sum(d[k] for d in data) or 1 for k in (1, 2, 3))
print(f"total warp-inst {ti:.4g}  avg threads {tt / ti:.1f}")
for name, lo, hi in regions:
    s = [d for d in data if lo <= d[0] <= hi]
    i, t, st = (sum(d[k] for d in s) for k in (1, 2, 3))
    print(f"  {name:16s} inst {100 * i / ti:5.1f}%  threads/inst {t / max(i, 1):5.1f}  stalls {100 * st / ts:5.1f}%")
