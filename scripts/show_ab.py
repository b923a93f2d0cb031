"""Print the A/B lines written by scripts/gpu_ab_env.sh: env, step ms, per-kernel ms."""
import json
import sys
from pathlib import Path

tag = sys.argv[1]
out = Path(__file__).resolve().parents[1] / "gpurun_out"
for line in (out / f"ab_{tag}_index.txt").read_text().splitlines():
    i, _, env = line.partition(" ")
    try:
        d = json.loads((out / f"ab_{tag}_{i}.json").read_text())
        print(f"{env or 'default':40s} step {d['ms_per_step']:9.2f} ms  " +
              "  ".join(f"{k} {v:8.2f}" for k, v in d.get("kernels_ms", {}).items()))
    except Exception as e:  # noqa: BLE001
        print(f"{env or 'default':40s} failed: {e}")
