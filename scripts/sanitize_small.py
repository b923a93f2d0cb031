"""compute-sanitizer target: one small sliced-mode batch (40 apps) and one
main-mode batch (300 apps) through gd_grid_select, checked against the oracle.

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_small.py
"""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2004_08177_b200 as gd
from paper_2004_08177_b200 import workload as W
import oracle_lib as O
for n, cl in ((40, "gtx980"), (300, "gtx980")):
    sc = W.make_scenario("san", n, cl, 40, 8, seed=5, w_clk=0.15)
    ctx = gd.Context(0)
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    budgets = np.full(sc.grid.n_apps, 1e9)
    got, e, t = gd.grid_select(me, mt, sc.grid, budgets, return_predictions=True)
    want, we, wt = O.oracle_grid(sc.energy, sc.time, sc.grid, budgets)
    print(n, np.array_equal(e.view(np.int64), we.view(np.int64)), np.array_equal(t.view(np.int64), wt.view(np.int64)))
