"""Where the end-to-end (host-buffer) time goes: H2D bandwidth, fixed per-call
overhead and the device-resident step, for configs[1] and the 64-app stream."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2004_08177_b200 as gd  # noqa: E402
from paper_2004_08177_b200 import workload as W  # noqa: E402

sc = W.make_scenario("e2e", 10000, "gtx980", 500, 8, seed=1234)
ctx = gd.Context(0)
me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
g = sc.grid
opts = gd.SchedulerOptions(budget="full")


def timeit(fn, n=30, w=5):
    for _ in range(w):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


for A in (10000, 64):
    hg = W.GridInputs(pin(g.rows[:A]), pin(g.cat_t[:A]), pin(g.cat_cols.astype(np.int32)), pin(g.sm), pin(g.mem),
                      g.sm_col, g.mem_col)
    hb = pin(np.ones(A))
    out = np.zeros(A, gd.DECISION_DTYPE)
    e2e = timeit(lambda: gd.grid_select(me, mt, hg, hb, opts, out=out))
    x = torch.from_numpy(hg.rows)
    d = torch.empty_like(x, device="cuda")
    torch.cuda.synchronize()
    h2d = timeit(lambda: (d.copy_(x, non_blocking=True), torch.cuda.synchronize()))
    ctx.set_timing(True)
    gd.grid_select(me, mt, hg, hb, opts, out=out)
    ks = ctx.kernel_times()
    ctx.set_timing(False)
    print(f"A={A}: e2e {e2e:.3f} ms | H2D rows {h2d:.3f} ms ({x.numel() * 8 / h2d / 1e6:.1f} GB/s) | "
          f"kernels {sum(v for _, v in ks):.3f} ms {[(k, round(v, 3)) for k, v in ks]}")
