#!/usr/bin/env python
"""Copy the ncu / bench evidence of one GPU run from gpurun_out/ into profiles/.

    python scripts/make_profiles.py <gpurun tag> <round tag> [config]

Writes profiles/<round>_launches.csv (per-kernel launch list: count, mean
duration, DRAM bytes, share of GPU time), profiles/<round>_grid_kernel.txt
(ncu --set full summary, per-source-line and per-opcode breakdown of the grid
kernel), profiles/<round>_bench.json (both bench arms) and updates
profiles/ncu_traffic.json (DRAM bytes per grid_acc_kernel launch -- the
dominant kernel -- from the --set full capture, read by bench.py for
roofline.traffic).
"""
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"


def launches(tag, rnd):
    rows = [r for r in csv.DictReader(l for l in open(OUT / f"launches_{tag}.csv") if not l.startswith("=="))]
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows:
        # kernel + grid size: the 10k-app grid launches and the 64-app
        # latency-stream launches of the same kernel are listed apart
        k = f'{r["Kernel Name"][:90]} grid{r["Grid Size"].replace(" ", "")}'

        agg[k][r["Metric Name"]] += float(r["Metric Value"])
        if r["Metric Name"] == "gpu__time_duration.sum":
            cnt[k] += 1
    total = sum(v["gpu__time_duration.sum"] for v in agg.values())
    with open(PROF / f"{rnd}_launches.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "mean_duration_us", "dram_read_bytes_per_launch",
                    "dram_write_bytes_per_launch", "share_of_gpu_time"])
        for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
            n = cnt[k]
            w.writerow([k, n, round(v["gpu__time_duration.sum"] / n / 1e3, 2),
                        int(v.get("dram__bytes_read.sum", 0) / n), int(v.get("dram__bytes_write.sum", 0) / n),
                        round(v["gpu__time_duration.sum"] / total, 4)])


def report(tag):
    for name in (f"prof_grid_{tag}.ncu-rep", f"prof_{tag}.ncu-rep"):
        if (OUT / name).exists():
            return OUT / name
    return None


def full_traffic(tag):
    """DRAM read+write bytes of one grid_acc_kernel launch (the dominant kernel)
    from the ncu --set full capture."""
    rep = report(tag)
    if rep is None:
        return None
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        if "grid_acc_kernel" in r[hdr.index("Kernel Name")]:
            tot = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(m)
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i]]
                tot += float(r[i].replace(",", "")) * scale
            return int(tot)
    return None


def kernel_summary(tag, rnd):
    rep = report(tag)
    parts = []
    for cmd in (["python", "scripts/ncu_summary.py", str(rep), "--raw",
                 r"dram__bytes_(read|write)\.sum$|lts__t_bytes\.sum$|l1tex__t_sector_hit_rate\.pct$|"
                 r"smsp__inst_executed_pipe_fp64|sm__pipe_fp64_cycles_active|"
                 r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared\.sum$|smsp__pcsamp_warps_issue_stalled_[a-z_]+$"],
                ["python", "scripts/ncu_lines.py", str(rep), "--top", "30", "--kernel", "acc"],
                ["python", "scripts/ncu_lines.py", str(rep), "--top", "30", "--kernel", "walk"],
                ["python", "scripts/ncu_sass.py", str(rep), "--top", "0", "--kernel", "acc"],
                ["python", "scripts/ncu_sass.py", str(rep), "--top", "0", "--kernel", "walk"]):
        parts.append("$ " + " ".join(cmd[1:]) + "\n" + subprocess.run(cmd, capture_output=True, text=True,
                                                                          cwd=ROOT).stdout)
    (PROF / f"{rnd}_grid_kernel.txt").write_text("\n".join(parts))


def main():
    tag, rnd = sys.argv[1], sys.argv[2]
    config = sys.argv[3] if len(sys.argv) > 3 else "c4"
    PROF.mkdir(exist_ok=True)
    launches(tag, rnd)
    traffic = full_traffic(tag)
    if report(tag) is not None:
        kernel_summary(tag, rnd)
    bench = {}
    for name in (f"bench_{tag}.json", f"bench_ref_{tag}.json"):
        p = OUT / name
        if p.exists() and p.read_text().strip():
            bench[name] = json.loads(p.read_text().strip().splitlines()[-1])
    if bench:
        (PROF / f"{rnd}_bench.json").write_text(json.dumps(bench, indent=1))
    if traffic is not None:
        t = PROF / "ncu_traffic.json"
        d = json.loads(t.read_text()) if t.exists() else {}
        d[config] = traffic
        t.write_text(json.dumps(d, indent=1))
    print("traffic", traffic)


if __name__ == "__main__":
    main()
