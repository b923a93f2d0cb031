#!/usr/bin/env python
"""Per-CUDA-source-line instruction and stall totals from an ncu report.

    python scripts/ncu_lines.py report.ncu-rep [--top N] [--kernel REGEX]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
kern = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else None
kf = ["-k", f"regex:{kern}"] if kern else []
out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows, cur_file, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    try:
        ie = float(r[hdr.index("Instructions Executed", 2)] or 0)
        st = float(r[hdr.index("Warp Stall Sampling (All Samples)", 2)] or 0)
    except ValueError:
        continue
    rows.append((cur_file, int(r[0]), r[1].strip(), ie, st))
ti = sum(x[3] for x in rows); ts = sum(x[4] for x in rows)
print(f"total inst {ti:.4g}  stall samples {ts:.0f}")
print("-- by instructions")
for f, ln, src, ie, st in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"  {f}:{ln:<4} {100*ie/ti:5.1f}% inst {100*st/ts:5.1f}% stall | {src[:80]}")
print("-- by stalls")
for f, ln, src, ie, st in sorted(rows, key=lambda x: -x[4])[:top // 2]:
    print(f"  {f}:{ln:<4} {100*ie/ti:5.1f}% inst {100*st/ts:5.1f}% stall | {src[:80]}")
