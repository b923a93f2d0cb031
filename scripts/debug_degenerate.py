"""Debug helper: the degenerate-model grid cases of test_k2_degenerate_models_and_values, one at a time, with the first mismatching (app, clock)."""
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, dataclasses
import paper_2004_08177_b200 as gd
from paper_2004_08177_b200 import workload as W
import oracle_lib as O
sc = W.make_scenario("deg", 80, "gtx980", 24, 6, seed=31, w_clk=0.2)
fe, ft = sc.energy, sc.time
ctx = gd.Context(0)
empty = dataclasses.replace(fe, tree_offsets=np.zeros(1, np.int64), feature=np.zeros(0, np.int32), threshold=np.zeros(0), left=np.zeros(0, np.int32), right=np.zeros(0, np.int32), leaf_value=np.zeros(0))
n_extra = 5
off = np.concatenate([ft.tree_offsets, ft.tree_offsets[-1] + 1 + np.arange(n_extra, dtype=np.int64)])
leafy = dataclasses.replace(ft, tree_offsets=off, feature=np.concatenate([ft.feature, np.full(n_extra, -1, np.int32)]), threshold=np.concatenate([ft.threshold, np.zeros(n_extra)]), left=np.concatenate([ft.left, np.full(n_extra, -1, np.int32)]), right=np.concatenate([ft.right, np.full(n_extra, -1, np.int32)]), leaf_value=np.concatenate([ft.leaf_value, np.linspace(-1, 1, n_extra)]))
thr = fe.threshold.copy(); internal = np.nonzero(fe.feature >= 0)[0]; rng = np.random.default_rng(3)
thr[rng.choice(internal, 20, replace=False)] = np.nan
f7 = internal[fe.feature[internal] == 7]; thr[f7[::3]] = 0.0; thr[f7[1::3]] = -0.0
weird = dataclasses.replace(fe, threshold=thr)
rows = sc.grid.rows.copy(); rows[::7, 7] = 0.0; rows[1::7, 7] = -0.0; rows[2::9, 11] = np.nan; rows[3::9, 12] = np.inf; rows[4::9, 13] = -np.inf
for name, g in (("plain", sc.grid), ("weirdrows", W.GridInputs(rows, sc.grid.cat_t, sc.grid.cat_cols, sc.grid.sm, sc.grid.mem, W.SM_COL, W.MEM_COL))):
  for tag, e_f, t_f in (("fe,ft", fe, ft), ("empty,leafy", empty, leafy), ("weird,leafy", weird, leafy), ("weird,ft", weird, ft), ("fe,leafy", fe, leafy)):
    me, mt = gd.Model.from_forest(e_f, ctx), gd.Model.from_forest(t_f, ctx)
    b = np.ones(g.n_apps)
    want, we, wt = O.oracle_grid(e_f, t_f, g, b)
    got, ge, gt = gd.grid_select(me, mt, g, b, return_predictions=True)
    be = (ge.view(np.int64) != we.view(np.int64)); bt = (gt.view(np.int64) != wt.view(np.int64))
    print(name, tag, "E bad", int(be.sum()), "T bad", int(bt.sum()), "apps", np.nonzero(be.any(1) | bt.any(1))[0][:8])
