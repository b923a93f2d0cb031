"""configs[4] latency probe: the 64-job stream as in bench.py's c5_latency
(L2 warm, no flush), with per-interval device times from the timing hook
(h2d | rank | walk | acc | d2h) and the wall latency."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2004_08177_b200 as gd  # noqa: E402
from paper_2004_08177_b200 import workload as W  # noqa: E402

A, B = 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 64
sc = W.make_scenario("c5", A, "gtx980", 500, 8, seed=1234)
ctx = gd.Context(0)
me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
g = sc.grid
opts = gd.SchedulerOptions(budget="full")
wins = [(W.GridInputs(pin(g.rows[lo:lo + B]), pin(g.cat_t[lo:lo + B]), pin(g.cat_cols.astype(np.int32)), pin(g.sm),
                      pin(g.mem), g.sm_col, g.mem_col), pin(np.ones(B))) for lo in range(0, A - B + 1, B)][:64]
out = pin(np.zeros(B, gd.DECISION_DTYPE).view(np.uint8)).view(gd.DECISION_DTYPE)
lat = []
for k in range(330):
    gw, bw = wins[k % len(wins)]
    t0 = time.perf_counter()
    gd.grid_select(me, mt, gw, bw, opts, out=out)
    if k >= 30:
        lat.append(time.perf_counter() - t0)
lat = np.array(lat) * 1e6
ctx.set_timing(True)
spans = []
for k in range(100):
    gw, bw = wins[k % len(wins)]
    gd.grid_select(me, mt, gw, bw, opts, out=out)
    spans.append(dict(ctx.kernel_times()))
ctx.set_timing(False)
med = {k: round(float(np.median([s.get(k, 0) for s in spans])) * 1e3, 1) for k in spans[0]}
print(f"B={B}: wall p50 {np.percentile(lat, 50):.1f} us p99 {np.percentile(lat, 99):.1f} us | timed intervals (us) {med} "
      f"sum {sum(med.values()):.1f}")
