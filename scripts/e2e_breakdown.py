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


flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for A in (10000, 64, 1):
    hg = W.GridInputs(pin(g.rows[:A]), pin(g.cat_t[:A]), pin(g.cat_cols.astype(np.int32)), pin(g.sm), pin(g.mem),
                      g.sm_col, g.mem_col)
    hb = pin(np.ones(A))
    out = np.zeros(A, gd.DECISION_DTYPE)

    def call():
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gd.grid_select(me, mt, hg, hb, opts, out=out)
        return time.perf_counter() - t0

    for _ in range(5):
        call()
    e2e = 1e3 * float(np.median([call() for _ in range(30)]))
    ctx.set_timing(True)
    spans = []
    for _ in range(10):
        call()
        spans.append(ctx.kernel_times())
    ctx.set_timing(False)
    names = [k for k, _ in spans[0]]
    med = {k: float(np.median([dict(sp)[k] if k in dict(sp) else 0 for sp in spans])) for k in names}
    gpu = sum(med.values())
    x = torch.from_numpy(hg.rows)
    d = torch.empty_like(x, device="cuda")
    torch.cuda.synchronize()
    h2d = timeit(lambda: (d.copy_(x, non_blocking=True), torch.cuda.synchronize()))
    print(f"A={A}: e2e {e2e:.3f} ms | device span {gpu:.3f} ms {[(k, round(v, 3)) for k, v in med.items()]} | "
          f"host-side remainder {e2e - gpu:.3f} ms | torch H2D of rows alone {h2d:.3f} ms "
          f"({x.numel() * 8 / h2d / 1e6:.1f} GB/s)")
