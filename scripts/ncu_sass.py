#!/usr/bin/env python
"""Per-opcode and per-region breakdown of an ncu source page (SASS view).

    python scripts/ncu_sass.py report.ncu-rep [--top N] [--kernel REGEX] [--dump FILE]
"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
kern = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else None
kf = ["-k", f"regex:{kern}"] if kern else []
out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(out)) if r]
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hi]
rows = rows[hi:]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[1:] if len(r) == len(hdr) and r[0] != hdr[0]]
if "--dump" in sys.argv:
    with open(sys.argv[sys.argv.index("--dump") + 1], "w") as fh:
        for r in body:
            fh.write(f"{float(r[ix['Instructions Executed']] or 0):12.0f} {float(r[ix['Warp Stall Sampling (All Samples)']] or 0):6.0f}  {r[ix['Source']].strip()}\n")
ie, st, th = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"], ix["Avg. Threads Executed"]
tot_i = sum(float(r[ie] or 0) for r in body)
tot_s = sum(float(r[st] or 0) for r in body)
ops = collections.Counter()
stalls = collections.Counter()
for r in body:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    ops[op] += float(r[ie] or 0)
    stalls[op] += float(r[st] or 0)
print(f"total warp-instructions executed {tot_i:.4g}, stall samples {tot_s:.0f}")
for op, n in ops.most_common(25):
    print(f"   {op:<10} {n:12.4g} ({100*n/tot_i:5.1f}% inst)  stalls {100*stalls[op]/max(tot_s,1):5.1f}%")
print("-- hottest SASS lines by stall samples")
for i, r in sorted(enumerate(body), key=lambda x: -float(x[1][st] or 0))[:top]:
    print(f"   [{i:5d}] {float(r[st] or 0):7.0f} st {float(r[ie] or 0):10.4g} ex {float(r[th] or 0):5.1f}thr  {r[ix['Source']].strip()[:90]}")
