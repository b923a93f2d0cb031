"""compute-sanitizer target: small batches through gd_grid_select covering
the sliced accumulate (40 apps), the main accumulate with 16-bit 512-app walk
tiles (300 apps), 8-bit 1024-app walk tiles (1500 apps, GDVFS_WIDE=2),
several batches with streamed inputs, a single-memory-clock catalog (folded
walk nodes), blocking and lazy stage refills and the device-buffer path -- each checked against the oracle.

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_small.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle_lib as O  # noqa: E402
import paper_2004_08177_b200 as gd  # noqa: E402
from paper_2004_08177_b200 import workload as W  # noqa: E402

ctx = gd.Context(0)
cases = [(40, {}), (300, {}), (1500, {"GDVFS_WIDE": "2"}),
         (3000, {"GDVFS_BATCH_BYTES": "3000000", "GDVFS_WIDE": "2"}), (300, {"FOLD": "1"}),
         (1500, {"GDVFS_LAZY": "0"}), (600, {"GDVFS_LAZY": "2", "GDVFS_WALK_BUFS": "3", "GDVFS_WIDE": "1"})]
for n, env in cases:
    os.environ.update({k: v for k, v in env.items() if k.startswith("GDVFS")})
    sc = W.make_scenario("san", n, "gtx980", 40, 8, seed=5, w_clk=0.15)
    g = sc.grid
    if "FOLD" in env:  # one memory clock: the walk folds those tests
        keep = g.mem == 3505
        g = W.GridInputs(g.rows, g.cat_t, g.cat_cols, g.sm[keep], g.mem[keep], g.sm_col, g.mem_col)
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    budgets = np.full(g.n_apps, 1e9)
    got, e, t = gd.grid_select(me, mt, g, budgets, return_predictions=True)
    want, we, wt = O.oracle_grid(sc.energy, sc.time, g, budgets)
    print(n, env, np.array_equal(e.view(np.int64), we.view(np.int64)), np.array_equal(t.view(np.int64), wt.view(np.int64)),
          flush=True)
    for k in env:
        os.environ.pop(k, None)
