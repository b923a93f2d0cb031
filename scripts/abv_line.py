"""One-line summary of a bench JSON line read from stdin (scripts/gpu_abv.sh)."""
import json
import sys

try:
    d = json.loads(sys.stdin.read().splitlines()[-1])
    k = d.get("kernels_ms", {})
    print(f"{d['ms_per_step']:.3f} ms  walk {k.get('walk', 0):.3f} acc {k.get('acc', 0):.3f}  "
          f"ok={d.get('device_vs_e2e_decisions_identical')}")
except Exception as e:  # noqa: BLE001
    print("failed:", e)
