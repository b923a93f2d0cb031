"""Debug helper: compare the grid kernel with the oracle on one scenario and
print the mismatch pattern (apps, clocks, magnitudes)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_lib as O  # noqa: E402
import paper_2004_08177_b200 as gd  # noqa: E402
from paper_2004_08177_b200 import workload as W  # noqa: E402

n_apps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
trees = int(sys.argv[2]) if len(sys.argv) > 2 else 60
w_clk = float(sys.argv[3]) if len(sys.argv) > 3 else 0.04
sc = W.make_scenario("dbg", n_apps, "gtx980", trees, 8, seed=11, w_clk=w_clk)
ctx = gd.Context(0)
me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
b = np.ones(n_apps)
_, ge, gt = gd.grid_select(me, mt, sc.grid, b, return_predictions=True)
_, we, wt = O.oracle_grid(sc.energy, sc.time, sc.grid, b)
for name, g, w in (("E", ge, we), ("T", gt, wt)):
    bad = g.view(np.int64) != w.view(np.int64)
    print(name, "mismatches", int(bad.sum()), "of", bad.size)
    if bad.any():
        apps = np.nonzero(bad.any(axis=1))[0]
        print("  apps", apps[:20], "clocks of first", np.nonzero(bad[apps[0]])[0][:40])
        a = apps[0]
        c = np.nonzero(bad[a])[0][:5]
        print("  got", g[a, c], "want", w[a, c])
