"""Print the key fields of bench JSON lines (gpurun_out/bench_*.json)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        lines = [l for l in open(path).read().splitlines() if l.startswith("{")]
        d = json.loads(lines[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable", e)
        continue
    br = d.get("binding_roofline", {})
    print(path, d.get("config", {}).get("workload", "")[:60])
    print(f"  value {d.get('value', 0):.4g} ms/step {d.get('ms_per_step', 0):.3f} kernels {d.get('kernels_ms')} "
          f"fp64 frac {br.get('frac', 0):.3f} e2e {d.get('e2e', {}).get('ms_per_step', 0):.2f} ms "
          f"consistent {d.get('device_vs_e2e_decisions_identical')} cpu {d.get('cpu_baseline', {}).get('value')}")
    for k, v in (d.get("extra_configs") or {}).items():
        print("  extra", k, {kk: v.get(kk) for kk in ("value", "ms_per_step", "kernels_ms", "p50_us", "p99_us", "error")})
