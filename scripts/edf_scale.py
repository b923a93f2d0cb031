"""remaining_time scheduling at scale: the EDF loop answering
every job by an O(C) scan vs by binary search on the GPU selection frontier,
on configs[1]-shaped tables (10k jobs x 267 clocks); decisions must match."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import oracle_lib as O  # noqa: E402
import paper_2004_08177_b200 as gd  # noqa: E402
from paper_2004_08177_b200 import workload as W  # noqa: E402

sc = W.make_scenario("edf", 10000, "gtx980", 500, 8, seed=1234)
ctx = gd.Context(0)
me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
_, E, T = gd.grid_select(me, mt, sc.grid, np.ones(sc.grid.n_apps), return_predictions=True)
rng = np.random.default_rng(5)
n = sc.grid.n_apps
jobs = np.zeros(n, O.JOB_DTYPE)
jobs["arrival_s"] = np.sort(rng.uniform(0, 40.0, size=n))
jobs["deadline_s"] = np.median(T, axis=1) * rng.uniform(1.0, 3.0, size=n)
jobs["app_rank"] = np.arange(n)
jobs["app_index"] = np.arange(n)
X = T * 0.01
opts = gd.SchedulerOptions()  # text, remaining_time, energy
t0 = time.perf_counter()
a, ao = gd.schedule_d_dvfs(jobs, E, T, sc.grid.sm, X, opts)
t_scan = time.perf_counter() - t0
t0 = time.perf_counter()
front = gd.frontier(E, T, sc.grid.sm, "energy", ctx=ctx)
t_front = time.perf_counter() - t0
t0 = time.perf_counter()
b, bo = gd.schedule_d_dvfs(jobs, E, T, sc.grid.sm, X, opts, front=front)
t_query = time.perf_counter() - t0
same = bool(np.array_equal(a.view(np.uint8), b.view(np.uint8)) and np.array_equal(ao, bo))
print(f"{n} jobs x {T.shape[1]} clocks, remaining_time/text: scan EDF {t_scan * 1e3:.2f} ms | frontier "
      f"{t_front * 1e3:.2f} ms (GPU, incl. H2D/D2H) + EDF {t_query * 1e3:.2f} ms | identical {same} | "
      f"scheduled {int((a['status'] == 0).sum())}")
