"""Walk-kernel per-CTA timeline for one configs[4] batch (needs a library
built with -DGD_WALK_TRACE, selected through GDVFS_LIB)."""
import ctypes as Ct
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2004_08177_b200 as gd  # noqa: E402
from paper_2004_08177_b200 import _capi  # noqa: E402
from paper_2004_08177_b200 import workload as W  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sc = W.make_scenario("c5", 4096, "gtx980", 500, 8, seed=1234)
ctx = gd.Context(0)
me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
g = sc.grid
gw = W.GridInputs(g.rows[:B], g.cat_t[:B], g.cat_cols.astype(np.int32), g.sm, g.mem, g.sm_col, g.mem_col)
opts = gd.SchedulerOptions(budget="full")
for _ in range(20):
    gd.grid_select(me, mt, gw, np.ones(B), opts)
buf = np.zeros((4096, 8), np.uint64)
lib = _capi.lib()
lib.gd_debug_walk_trace.argtypes = [Ct.c_void_p, Ct.c_int]
lib.gd_debug_walk_trace(buf.ctypes.data, 4096)
used = buf[:, 0] > 0
t = buf[used].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
print(f"CTAs {used.sum()}: start spread {rel[:, 0].max():.2f} us; end (max t5) {rel[:, 5].max():.2f} us")
for k, name in enumerate(["start", "init+produce", "ranks", "stage0 ready", "walks done", "jobs done"]):
    col = rel[:, k]
    print(f"  {name:14s} median {np.median(col):7.2f} p90 {np.percentile(col, 90):7.2f} max {col.max():7.2f} us")
d = np.diff(rel[:, :6], axis=1)
for k, name in enumerate(["init+produce", "ranks", "TMA wait", "walks", "jobs"]):
    print(f"  delta {name:12s} median {np.median(d[:, k]):6.2f} p90 {np.percentile(d[:, k], 90):6.2f} max {d[:, k].max():6.2f}")
slow = np.argsort(-d[:, 3])[:12]
idx = np.nonzero(used)[0]
print("slowest walk phases (cta: walks us, jobs us):", [(int(idx[i]), round(float(d[i, 3]), 2), round(float(d[i, 4]), 2)) for i in slow])
