"""GPU parity: the sm_100a kernels, called through the C ABI, against the oracle
and the reference's golden vectors.  Integer/index results (leaf ids, chosen
clocks, statuses) must be identical; predictions are compared bit-for-bit
(the path is exact FP64 -- stricter than north_star's 1e-5 relative bound,
which tests/test_gpu_parity.py::test_sum_tolerance_statement documents).
"""
import itertools
import os

import numpy as np
import pytest

import oracle_lib as O
import paper_2004_08177_b200 as gd
from helpers import GOLDEN, bits, c1_combo, c1_small, decisions_equal, golden_forest, parse_model_text, tie_tables
from paper_2004_08177_b200 import workload as W

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5  # north_star's bound for summed predictions; we require 0 ulp


@pytest.fixture(scope="module")
def ctx():
    c = gd.Context(0)
    yield c
    c.close()


def opts_of(mode, budget, obj, be):
    return gd.SchedulerOptions(mode=["text", "literal"][mode], budget=["remaining", "full"][budget],
                               objective=["energy", "power"][obj], best_effort_fallback=bool(be))


# ---- K1 predict_rows ---------------------------------------------------------

@pytest.mark.parametrize("key", ["complete_0", "complete_1", "irregular_0", "irregular_1", "neg"])
def test_k1_predict_matches_reference_golden(ctx, key):
    npz = np.load(GOLDEN / "predict.npz")
    f = golden_forest(npz, key, 1 if key.endswith("_1") else 0)
    m = gd.Model.from_forest(f, ctx)
    got, ids = m.predict(npz[f"{key}_rows"], leaf_ids=True)
    assert np.array_equal(bits(got), bits(npz[f"{key}_pred"]))
    want_p, want_ids = O.oracle_predict(f, npz[f"{key}_rows"], leaf_ids=True)
    assert np.array_equal(ids, want_ids)


@pytest.mark.parametrize("form", ["auto", "rows_on_lanes", "trees_on_lanes"])
@pytest.mark.parametrize("leaf_prob,depth,trees", [(0.0, 8, 67), (0.35, 10, 40), (0.0, 1, 5), (0.2, 12, 33)])
def test_k1_predict_leaf_ids_vs_oracle(ctx, leaf_prob, depth, trees, form, monkeypatch):
    # both K1 forms (the library picks by batch size; forced here): 350 rows =
    # 10 full 32-row tiles + a partial one; odd tree counts hit the lockstep tail
    if form != "auto":
        monkeypatch.setenv("GDVFS_K1_TREES_ON_LANES", "1" if form == "trees_on_lanes" else "0")
    sc = W.make_scenario("k1", 50, "gtx980", trees, depth, seed=depth, w_clk=0.1, leaf_prob=leaf_prob)
    rows = np.repeat(sc.grid.rows, 7, axis=0)
    rows[:, W.SM_COL] = np.resize(sc.grid.sm, rows.shape[0])
    for f in (sc.energy, sc.time):
        m = gd.Model.from_forest(f, ctx)
        got, ids = m.predict(rows, leaf_ids=True)
        want, want_ids = O.oracle_predict(f, rows, leaf_ids=True)
        assert np.array_equal(bits(got), bits(want))
        assert np.array_equal(ids, want_ids)


def test_k1_model_file_and_c1_models(ctx):
    npz = np.load(GOLDEN / "model_file_pred.npz")
    m = gd.Model.load_file(GOLDEN / "model_time_small.txt", ctx)
    assert np.array_equal(bits(m.predict(npz["rows"])), bits(npz["pred"]))
    s = c1_small()
    me = gd.Model.load_file(s["model_energy"], ctx)
    rows = s["rows"]
    got, ids = me.predict(rows, leaf_ids=True)
    want, want_ids = O.oracle_predict(s["fe"], rows, leaf_ids=True)
    assert np.array_equal(bits(got), bits(want)) and np.array_equal(ids, want_ids)


def test_k1_edge_cases(ctx):
    f = W.make_scenario("e", 3, "p100", 5, 3, seed=2).time
    m = gd.Model.from_forest(f, ctx)
    assert m.predict(np.zeros((0, W.N_COLS))).shape == (0,)
    with pytest.raises(ValueError, match="column mismatch"):
        m.predict(np.zeros((2, W.N_COLS - 1)))
    # zero trees: base prediction only (models.cpp:370-377 with an empty loop)
    z = W.Forest(np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0), np.zeros(0, np.int32),
                 np.zeros(0, np.int32), np.zeros(0), 3.5, 0.1, 1, W.N_COLS)
    out = gd.Model.from_forest(z, ctx).predict(np.ones((4, W.N_COLS)))
    assert np.all(out == 3.5)
    # a single-leaf tree
    one = W.Forest(np.array([0, 1], np.int64), np.array([-1], np.int32), np.zeros(1), np.array([-1], np.int32),
                   np.array([-1], np.int32), np.array([2.0]), 1.0, 0.5, 1, W.N_COLS)
    assert np.all(gd.Model.from_forest(one, ctx).predict(np.ones((3, W.N_COLS))) == 2.0)


def test_k1_linear(ctx):
    rng = np.random.default_rng(0)
    coef = rng.normal(size=W.N_COLS)
    rows = rng.normal(size=(300, W.N_COLS)) * 10
    for target in (0, 1):
        m = gd.Model.linear(coef, -0.25, target=target, ctx=ctx)
        got = m.predict(rows)
        want = O.oracle_predict_linear(coef, -0.25, int(target == 0), rows)
        assert np.array_equal(bits(got), bits(want))


# ---- K2+K3 fused grid --------------------------------------------------------

SCENARIOS = {
    "c2_shape": dict(n_apps=300, catalog="gtx980", n_trees=60, depth=8, w_clk=0.04),
    "stress_clk": dict(n_apps=200, catalog="gtx980", n_trees=40, depth=8, w_clk=0.25),
    "fallback": dict(n_apps=64, catalog="b200", n_trees=35, depth=10, w_clk=0.6),
    "irregular": dict(n_apps=150, catalog="p100", n_trees=70, depth=10, w_clk=0.05, leaf_prob=0.3),
    "tiny_grid": dict(n_apps=33, catalog="p100", n_trees=3, depth=2, w_clk=0.5),
}


def scenario(name):
    kw = dict(SCENARIOS[name])
    return W.make_scenario(name, kw.pop("n_apps"), kw.pop("catalog"), kw.pop("n_trees"), kw.pop("depth"), seed=11,
                           **kw)


@pytest.mark.parametrize("sliced", ["0", "1"])
@pytest.mark.parametrize("name", list(SCENARIOS))
def test_k2_grid_predictions_and_decisions_vs_oracle(ctx, name, sliced, monkeypatch):
    # both accumulate layouts: warp pair per app, and per (app, clock slice)
    monkeypatch.setenv("GDVFS_ACC_SLICED", sliced)
    sc = scenario(name)
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    _, e0, t0 = O.oracle_grid(sc.energy, sc.time, sc.grid, np.ones(sc.grid.n_apps))
    budgets = W.deadlines_from_times(t0, seed=5)
    for combo in itertools.product((0, 1), (1,), (0, 1), (0, 1)):
        mode, _, obj, be = combo
        want, we, wt = O.oracle_grid(sc.energy, sc.time, sc.grid, budgets, mode, obj, be)
        got, ge, gt = gd.grid_select(me, mt, sc.grid, budgets, opts_of(*combo), return_predictions=True)
        assert np.array_equal(bits(ge), bits(we)), (name, combo)
        assert np.array_equal(bits(gt), bits(wt)), (name, combo)
        assert decisions_equal(got, want), (name, combo)


def test_k2_graph_replay_stream_vs_oracle(ctx):
    """Decisions-only small calls are captured once per shape and replayed as
    a CUDA graph (the configs[4] stream): successive windows, both selection
    modes, a buffer-growing large call in between (the captured addresses
    move: the graph must be rebuilt), and a second model pair."""
    sc = W.make_scenario("replay", 1200, "gtx980", 60, 8, seed=31, w_clk=0.08)
    g = sc.grid
    _, _, t0 = O.oracle_grid(sc.energy, sc.time, g, np.ones(g.n_apps))
    budgets = W.deadlines_from_times(t0, seed=3)

    def window(lo, n):
        return W.GridInputs(np.ascontiguousarray(g.rows[lo:lo + n]), np.ascontiguousarray(g.cat_t[lo:lo + n]),
                            g.cat_cols.astype(np.int32), g.sm.astype(np.int32), g.mem.astype(np.int32), g.sm_col,
                            g.mem_col), np.ascontiguousarray(budgets[lo:lo + n])

    # clock columns switched between two calls of one shape: the models' grid
    # nodes are recoded in place, so a graph captured for the first columns
    # must not be replayed for them afterwards
    me0, mt0 = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    gw, bw = window(0, 64)
    swapped = W.GridInputs(gw.rows, gw.cat_t, gw.cat_cols, gw.sm, gw.mem, g.mem_col, g.sm_col)
    for grid_in in (gw, gw, swapped, gw, swapped, gw):
        got = gd.grid_select(me0, mt0, grid_in, bw, opts_of(0, 1, 0, 0))
        want, _, _ = O.oracle_grid(sc.energy, sc.time, grid_in, bw, 0, 0, 0)
        assert decisions_equal(got, want)
    other = W.make_scenario("replay2", 8, "gtx980", 45, 7, seed=77, w_clk=0.1)
    for pair in range(2):
        f_e, f_t = (sc.energy, sc.time) if pair == 0 else (other.energy, other.time)
        me, mt = gd.Model.from_forest(f_e, ctx), gd.Model.from_forest(f_t, ctx)
        for combo in [(0, 1, 0, 0), (1, 1, 1, 1)]:
            mode, _, obj, be = combo
            for k, n in enumerate([64, 64, 64, 1000, 64, 64]):
                gw, bw = window((k * 64) % 200, n)
                got = gd.grid_select(me, mt, gw, bw, opts_of(*combo))
                want, _, _ = O.oracle_grid(f_e, f_t, gw, bw, mode, obj, be)
                assert decisions_equal(got, want), (pair, combo, k)


def test_k2_graph_replay_n_records_change(ctx):
    """With rec_of_clock NULL the ABI allows n_records >= n_apps (record =
    app); the staged offsets of cat_t .. budgets depend on n_records, so a
    graph captured at one n_records must not be replayed at another (the
    replay key includes it).  Alternates R = A and R > A at the same A."""
    import ctypes as C

    from paper_2004_08177_b200 import _capi
    sc = W.make_scenario("nrec", 200, "gtx980", 40, 8, seed=41, w_clk=0.08)
    g = sc.grid
    A = 64
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    _, _, t0 = O.oracle_grid(sc.energy, sc.time, g, np.ones(g.n_apps))
    budgets = np.ascontiguousarray(W.deadlines_from_times(t0, seed=4)[:A])
    sub = W.GridInputs(np.ascontiguousarray(g.rows[:A]), np.ascontiguousarray(g.cat_t[:A]), g.cat_cols, g.sm, g.mem,
                       g.sm_col, g.mem_col)
    want, _, _ = O.oracle_grid(sc.energy, sc.time, sub, budgets, 0, 0, 0)
    cat_cols, sm, mem = (np.ascontiguousarray(x, np.int32) for x in (g.cat_cols, g.sm, g.mem))
    opts = opts_of(0, 1, 0, 0).opts()
    for R in (A, 100, A, A, 150, 150, A, 100):
        rows = np.ascontiguousarray(g.rows[:R])
        cat = np.ascontiguousarray(g.cat_t[:R])
        gs = _capi.Grid(gd._ptr(rows), R, rows.shape[1], cat.shape[1], gd._ptr(cat), gd._ptr(cat_cols), None, A,
                        gd._ptr(sm), gd._ptr(mem), sm.shape[0], g.sm_col, g.mem_col, 0, gd._ptr(budgets))
        out = np.zeros(A, gd.DECISION_DTYPE)
        gd._raise(_capi.lib().gd_grid_select(ctx.handle, me.handle, mt.handle, C.byref(gs), C.byref(opts),
                                             gd._ptr(out), None, None))
        assert decisions_equal(out, want), R


@pytest.mark.parametrize("seed", range(64))
def test_k2_fuzz_catalogs_and_shapes_vs_oracle(ctx, seed):
    """Random catalogs (any size up to 512, 1..40 memory clocks, arbitrary
    order or the reference's (mem, sm) order, duplicate pairs allowed -- the
    reference only ever sees unique sorted catalogs; for the others the
    oracle's per-index semantics are the contract),
    random tree shapes / clock-split rates, batch sizes on both sides of the
    latency-mode switch, random selection options: predictions and decisions
    bit-identical to the oracle, with and without the E/T tables (the
    decisions-only calls also exercise the graph replay)."""
    rng = np.random.default_rng(1000 + seed)
    C = int(rng.choice([1, 2, 5, 31, 32, 33, 64, 100, 267, 300, 512]))
    n_mem = int(rng.integers(1, min(C, 40) + 1))
    mems = rng.choice(np.arange(300, 9000, 7), size=n_mem, replace=False)
    sm = rng.integers(100, 2500, size=C).astype(np.int32)
    mem = rng.choice(mems, size=C).astype(np.int32)
    if rng.random() < 0.5:
        order = np.lexsort((sm, mem))
        sm, mem = sm[order], mem[order]
    n_apps = int(rng.choice([1, 7, 64, 255, 257, 600]))
    sc = W.make_scenario("fuzz", n_apps, (sm, mem), int(rng.integers(1, 80)), int(rng.integers(1, 11)), seed=seed,
                         w_clk=float(rng.choice([0.0, 0.05, 0.2, 0.5])), leaf_prob=float(rng.choice([0.0, 0.3])))
    if rng.random() < 0.5:  # NaN / extreme feature values (clock columns are substituted anyway)
        rows = sc.grid.rows
        rows[rng.random(rows.shape) < 0.03] = np.nan
        rows[rng.random(rows.shape) < 0.01] = 1e300
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    _, _, t0 = O.oracle_grid(sc.energy, sc.time, sc.grid, np.ones(n_apps))
    budgets = W.deadlines_from_times(t0, seed=seed)
    for _ in range(2):
        combo = tuple(int(x) for x in rng.integers(0, 2, size=4))
        mode, _, obj, be = combo
        want, we, wt = O.oracle_grid(sc.energy, sc.time, sc.grid, budgets, mode, obj, be)
        got, ge, gt = gd.grid_select(me, mt, sc.grid, budgets, opts_of(*combo), return_predictions=True)
        assert np.array_equal(bits(ge), bits(we)) and np.array_equal(bits(gt), bits(wt)), (seed, combo)
        assert decisions_equal(got, want), (seed, combo)
        for _ in range(2):
            assert decisions_equal(gd.grid_select(me, mt, sc.grid, budgets, opts_of(*combo)), want), (seed, combo)


# Internal paths of the walk / accumulate pipeline forced through knobs (the
# library reads them per call): several batches, small shared-memory windows
# (walks continue from global memory), residue-table pool overflow (FULL
# records), deeper buffer rings, one app group per CTA.
KNOBS = {
    "batches": {"GDVFS_BATCH_BYTES": "300000"},
    "windowed": {"GDVFS_WIN_NODES": "16"},
    "pool_overflow": {"GDVFS_POOL_DIV": "1000000"},
    "ring4": {"GDVFS_WALK_BUFS": "4"},
    "one_group": {"GDVFS_WALK_GROUPS": "1", "GDVFS_WALK_BUFS": "3"},
    "sliced_acc": {"GDVFS_ACC_SLICED": "1"},
    "wide_tiles": {"GDVFS_WIDE": "2"},
    "narrow_tiles": {"GDVFS_WIDE": "0"},
    "split_major": {"GDVFS_WALK_SPLIT_MAJOR": "1", "GDVFS_WALK_SPLITS": "7"},
    "tile_major": {"GDVFS_WALK_SPLIT_MAJOR": "0", "GDVFS_WALK_SPLITS": "3"},
    "res_levels_3": {"GDVFS_RES_LEVELS": "3"},
    "res_levels_4": {"GDVFS_RES_LEVELS": "4"},
    "res_levels_1": {"GDVFS_RES_LEVELS": "1"},
    "subs2": {"GDVFS_WALK_SUBS": "2"},
    "lazy_refill": {"GDVFS_LAZY": "2", "GDVFS_WALK_BUFS": "3"},
    "blocking_refill": {"GDVFS_LAZY": "0"},
    "job_runs_32": {"GDVFS_JOB_RUN": "32"},
    "job_runs_96_lazy": {"GDVFS_JOB_RUN": "96", "GDVFS_LAZY": "2"},
}


@pytest.mark.parametrize("levels", ["5", "4"])
@pytest.mark.parametrize("w_clk,depth", [(0.25, 11), (0.4, 9), (0.15, 12)])
def test_k2_deep_residues_tables4_and_full(ctx, w_clk, depth, levels, monkeypatch):
    # clock-heavy deep trees: residues with 3-5 test levels (TABLE / TABLE4 /
    # TABLE5 records) and deeper ones (FULL), in both accumulate modes, with
    # tables up to 5 or up to 4 levels
    monkeypatch.setenv("GDVFS_RES_LEVELS", levels)
    sc = W.make_scenario("deep_res", 300, "gtx980", 40, depth, seed=int(100 * w_clk) + depth, w_clk=w_clk)
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    _, _, t0 = O.oracle_grid(sc.energy, sc.time, sc.grid, np.ones(sc.grid.n_apps))
    budgets = W.deadlines_from_times(t0, seed=5)
    want, we, wt = O.oracle_grid(sc.energy, sc.time, sc.grid, budgets)
    for n in (300, 60):  # 60 apps: the sliced (latency) accumulate
        g = W.GridInputs(sc.grid.rows[:n], sc.grid.cat_t[:n], sc.grid.cat_cols, sc.grid.sm, sc.grid.mem,
                         sc.grid.sm_col, sc.grid.mem_col)
        got, ge, gt = gd.grid_select(me, mt, g, budgets[:n], return_predictions=True)
        assert np.array_equal(bits(ge), bits(we[:n])) and np.array_equal(bits(gt), bits(wt[:n]))
        assert decisions_equal(got, want[:n])


@pytest.mark.parametrize("knob", list(KNOBS))
def test_k2_internal_paths_vs_oracle(ctx, knob, monkeypatch):
    for k, v in KNOBS[knob].items():
        monkeypatch.setenv(k, v)
    sc = W.make_scenario(knob, 700, "gtx980", 90, 9, seed=23, w_clk=0.08)
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    _, _, t0 = O.oracle_grid(sc.energy, sc.time, sc.grid, np.ones(sc.grid.n_apps))
    budgets = W.deadlines_from_times(t0, seed=9)
    want, we, wt = O.oracle_grid(sc.energy, sc.time, sc.grid, budgets)
    got, ge, gt = gd.grid_select(me, mt, sc.grid, budgets, return_predictions=True)
    assert np.array_equal(bits(ge), bits(we)) and np.array_equal(bits(gt), bits(wt))
    assert decisions_equal(got, want)


def _forest_edit(f, **kw):
    import dataclasses
    return dataclasses.replace(f, **kw)


def test_k2_degenerate_models_and_values(ctx):
    # Models / rows at the edges of the contract: an ensemble with no trees
    # (prediction = base), single-leaf trees, NaN thresholds (never taken:
    # x <= NaN is false), NaN and +/-inf feature values (ranks at the ends),
    # duplicate thresholds and -0.0 / 0.0 on one feature.
    sc = W.make_scenario("deg", 80, "gtx980", 24, 6, seed=31, w_clk=0.2)
    fe, ft = sc.energy, sc.time
    empty = _forest_edit(fe, tree_offsets=np.zeros(1, np.int64), feature=np.zeros(0, np.int32),
                         threshold=np.zeros(0), left=np.zeros(0, np.int32), right=np.zeros(0, np.int32),
                         leaf_value=np.zeros(0))
    # single-leaf trees appended to the time model
    n_extra = 5
    off = np.concatenate([ft.tree_offsets, ft.tree_offsets[-1] + 1 + np.arange(n_extra, dtype=np.int64)])
    leafy = _forest_edit(ft, tree_offsets=off, feature=np.concatenate([ft.feature, np.full(n_extra, -1, np.int32)]),
                         threshold=np.concatenate([ft.threshold, np.zeros(n_extra)]),
                         left=np.concatenate([ft.left, np.full(n_extra, -1, np.int32)]),
                         right=np.concatenate([ft.right, np.full(n_extra, -1, np.int32)]),
                         leaf_value=np.concatenate([ft.leaf_value, np.linspace(-1, 1, n_extra)]))
    thr = fe.threshold.copy()
    internal = np.nonzero(fe.feature >= 0)[0]
    rng = np.random.default_rng(3)
    thr[rng.choice(internal, 20, replace=False)] = np.nan
    f7 = internal[fe.feature[internal] == 7]
    thr[f7[::3]] = 0.0
    thr[f7[1::3]] = -0.0
    weird = _forest_edit(fe, threshold=thr)
    rows = sc.grid.rows.copy()
    rows[::7, 7] = 0.0
    rows[1::7, 7] = -0.0
    rows[2::9, 11] = np.nan
    rows[3::9, 12] = np.inf
    rows[4::9, 13] = -np.inf
    g = W.GridInputs(rows, sc.grid.cat_t, sc.grid.cat_cols, sc.grid.sm, sc.grid.mem, W.SM_COL, W.MEM_COL)
    for e_f, t_f in ((empty, leafy), (weird, leafy), (weird, ft)):
        me, mt = gd.Model.from_forest(e_f, ctx), gd.Model.from_forest(t_f, ctx)
        _, _, t0 = O.oracle_grid(e_f, t_f, g, np.ones(g.n_apps))
        budgets = W.deadlines_from_times(t0, seed=4)
        want, we, wt = O.oracle_grid(e_f, t_f, g, budgets)
        got, ge, gt = gd.grid_select(me, mt, g, budgets, return_predictions=True)
        assert np.array_equal(bits(ge), bits(we)) and np.array_equal(bits(gt), bits(wt))
        assert decisions_equal(got, want)


@pytest.mark.parametrize("n_mem", [1, 4, 31, 32, 40])
def test_k2_clock_lane_maps(ctx, n_mem):
    # Catalogs whose memory-clock runs fit 32 lanes use the per-lane uniform
    # memory clock layout; more runs than lanes fall back to contiguous slots.
    rng = np.random.default_rng(n_mem)
    mems = np.sort(rng.choice(np.arange(300, 4000), size=n_mem, replace=False))
    per = max(1, 96 // n_mem)
    pairs = sorted({(int(sm), int(m)) for m in mems for sm in rng.choice(np.arange(300, 2000), size=per)},
                   key=lambda p: (p[1], p[0]))
    sm = np.array([p[0] for p in pairs], np.int32)
    mem = np.array([p[1] for p in pairs], np.int32)
    sc = W.make_scenario("map", 96, "gtx980", 40, 8, seed=n_mem, w_clk=0.3)
    cols = W._ColumnModel(np.random.default_rng(1), W.N_COLS, W.CAT_COLS, sm, mem, W.SM_COL, W.MEM_COL)
    fe = W.make_forest(cols, 40, 8, 0, 5, w_clk=0.3)
    ft = W.make_forest(cols, 40, 8, 1, 6, w_clk=0.3)
    g = W.GridInputs(sc.grid.rows, sc.grid.cat_t, sc.grid.cat_cols, sm, mem, W.SM_COL, W.MEM_COL)
    me, mt = gd.Model.from_forest(fe, ctx), gd.Model.from_forest(ft, ctx)
    _, _, t0 = O.oracle_grid(fe, ft, g, np.ones(g.n_apps))
    budgets = W.deadlines_from_times(t0, seed=2)
    for combo in ((0, 1, 0, 0), (1, 1, 1, 1)):
        want, we, wt = O.oracle_grid(fe, ft, g, budgets, combo[0], combo[2], combo[3])
        got, ge, gt = gd.grid_select(me, mt, g, budgets, opts_of(*combo), return_predictions=True)
        assert np.array_equal(bits(ge), bits(we)) and np.array_equal(bits(gt), bits(wt)), combo
        assert decisions_equal(got, want), combo


def test_k2_general_mode_c1_golden(ctx):
    # Per-clock records (nearest-record substitution, scheduler.cpp:341-359):
    # predictions must equal the reference's ClockPredictor outputs bit for bit.
    s = c1_small()
    me, mt = gd.Model.load_file(s["model_energy"], ctx), gd.Model.load_file(s["model_time"], ctx)
    got, e, t = gd.grid_select(me, mt, s["grid"], s["deadline"], gd.SchedulerOptions(budget="full"),
                               return_predictions=True)
    assert np.array_equal(bits(e), bits(s["pred_energy"]))
    assert np.array_equal(bits(t), bits(s["pred_time"]))
    want, _, _ = O.oracle_grid(s["fe"], s["ft"], s["grid"], s["deadline"])
    assert decisions_equal(got, want)


@pytest.mark.parametrize("tag", ["".join(map(str, c)) for c in itertools.product((0, 1), repeat=4)])
def test_end_to_end_schedule_c1_golden(ctx, tag):
    # GPU predictions -> host EDF loop == the reference's schedule_d_dvfs.
    s = c1_small()
    me, mt = gd.Model.load_file(s["model_energy"], ctx), gd.Model.load_file(s["model_time"], ctx)
    _, e, t = gd.grid_select(me, mt, s["grid"], s["deadline"], return_predictions=True)
    mode, budget, obj, be = (int(c) for c in tag)
    want, want_order = c1_combo(s, tag)
    got, order = gd.schedule_d_dvfs(s["jobs"], e, t, s["sm"], s["exec"], opts_of(mode, budget, obj, be))
    assert decisions_equal(got, want) and np.array_equal(order, want_order)


def test_c1_full_scale_live_reference(ctx, tmp_path):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    s = O.ref_c1_scenario(tmp_path, seed=7, iters=100, depth=10, n_jobs=100)
    me, mt = gd.Model.load_file(s["model_energy"], ctx), gd.Model.load_file(s["model_time"], ctx)
    g = W.GridInputs(s["rows"], s["cat_t"], s["cat_cols"], s["sm"], s["mem"], s["sm_col"], s["mem_col"],
                     s["rec_of_clock"])
    _, e, t = gd.grid_select(me, mt, g, s["deadline"], return_predictions=True)
    assert np.array_equal(bits(e), bits(s["pred_energy"])) and np.array_equal(bits(t), bits(s["pred_time"]))
    jobs = np.zeros(s["n_jobs"], O.JOB_DTYPE)
    jobs["arrival_s"], jobs["deadline_s"] = s["arrival"], s["deadline"]
    jobs["app_rank"] = jobs["app_index"] = np.arange(s["n_jobs"])
    got, order = gd.schedule_d_dvfs(jobs, e, t, s["sm"], s["exec"])
    assert decisions_equal(got, s["decisions"]) and np.array_equal(order, s["order"])


def test_k2_edge_cases(ctx):
    sc = scenario("tiny_grid")
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    # empty batch
    g0 = W.GridInputs(sc.grid.rows[:0], sc.grid.cat_t[:0], sc.grid.cat_cols, sc.grid.sm, sc.grid.mem, W.SM_COL,
                      W.MEM_COL)
    assert gd.grid_select(me, mt, g0, np.zeros(0)).shape == (0,)
    # single-clock catalog; all infeasible with and without best effort
    g1 = W.GridInputs(sc.grid.rows, sc.grid.cat_t, sc.grid.cat_cols, sc.grid.sm[:1], sc.grid.mem[:1], W.SM_COL,
                      W.MEM_COL)
    for be in (0, 1):
        want, _, _ = O.oracle_grid(sc.energy, sc.time, g1, np.full(sc.grid.n_apps, -1.0), 0, 0, be)
        got = gd.grid_select(me, mt, g1, np.full(sc.grid.n_apps, -1.0), opts_of(0, 1, 0, be))
        assert decisions_equal(got, want)
        assert np.all(got["status"] == (0 if be else 1))
    # budget exactly equal to a candidate's time is feasible (T > budget skips)
    _, _, t = O.oracle_grid(sc.energy, sc.time, sc.grid, np.ones(sc.grid.n_apps))
    b = t[:, 5].copy()
    want, _, _ = O.oracle_grid(sc.energy, sc.time, sc.grid, b)
    assert decisions_equal(gd.grid_select(me, mt, sc.grid, b), want)
    assert np.all(want["status"] == 0)
    # wrong model roles / column counts fail loudly
    with pytest.raises(ValueError):
        gd.grid_select(mt, me, sc.grid, b)
    bad = W.GridInputs(sc.grid.rows[:, :10], sc.grid.cat_t, sc.grid.cat_cols, sc.grid.sm, sc.grid.mem, 3, 4)
    with pytest.raises(ValueError):
        gd.grid_select(me, mt, bad, b)


# ---- K3 select alone -----------------------------------------------------------

@pytest.mark.parametrize("seed", range(4))
def test_k3_acceptance1_truth_golden(ctx, seed):
    # SPEC.md:599 acceptance #1: text selection on the truth tables == oracle_per_job.
    npz = np.load(GOLDEN / "truth.npz")
    got = gd.select(npz[f"s{seed}_E"], npz[f"s{seed}_T"], npz["sm"], npz[f"s{seed}_deadline"], ctx=ctx)
    assert decisions_equal(got, npz[f"s{seed}_decisions"])


@pytest.mark.parametrize("n_clocks", [1, 2, 31, 32, 33, 62, 200, 267, 512])
def test_k3_tie_breaks_vs_oracle(ctx, n_clocks):
    rng = np.random.default_rng(n_clocks)
    A = 257
    E, T = tie_tables(rng, A, n_clocks)
    sm = np.sort(rng.integers(100, 2000, size=n_clocks)).astype(np.int32)  # duplicates allowed (multi-mem grids)
    budgets = rng.choice(np.unique(T), size=A) + rng.choice([0.0, -0.1, 0.1], size=A)
    for combo in itertools.product((0, 1), (1,), (0, 1), (0, 1)):
        mode, _, obj, be = combo
        want = O.oracle_select(E, T, sm, budgets, mode, obj, be)
        got = gd.select(E, T, sm, budgets, opts_of(*combo), ctx=ctx)
        assert decisions_equal(got, want), combo


@pytest.mark.parametrize("n_clocks", [1, 2, 33, 62, 267, 512])
def test_frontier_kernel_vs_reference(ctx, n_clocks):
    from helpers import frontier_ref
    rng = np.random.default_rng(n_clocks)
    A = 40
    E, T = tie_tables(rng, A, n_clocks)
    E[5, 0] = np.inf
    sm = np.sort(rng.integers(100, 2000, size=n_clocks)).astype(np.int32)
    for obj in ("energy", "power"):
        ts, best, first = gd.frontier(E, T, sm, obj, ctx=ctx)
        wts, wbest, wfirst = frontier_ref(E, T, sm, int(obj == "power"))
        assert np.array_equal(bits(ts), bits(wts)) and np.array_equal(first, wfirst)
        ok = wfirst >= 0  # rows flagged non-finite are answered by a scan; their best[] is not used
        assert np.array_equal(best[ok], wbest[ok])


def test_remaining_time_edf_with_frontier_c1_golden(ctx):
    # The reference's default mode (remaining_time, text) answered from the
    # GPU frontier == the reference's schedule_d_dvfs decisions.
    s = c1_small()
    for tag in ("0000", "0010", "0001", "0011"):
        mode, budget, obj, be = (int(c) for c in tag)
        front = gd.frontier(s["pred_energy"], s["pred_time"], s["sm"], ["energy", "power"][obj], ctx=ctx)
        got, order = gd.schedule_d_dvfs(s["jobs"], s["pred_energy"], s["pred_time"], s["sm"], s["exec"],
                                        opts_of(mode, budget, obj, be), front=front)
        want, want_order = c1_combo(s, tag)
        assert decisions_equal(got, want) and np.array_equal(order, want_order), tag


def test_spec_examples_gpu(ctx):
    E, T = np.array([[100.0, 150.0]] * 3), np.array([[10.0, 5.0]] * 3)
    got = gd.select(E, T, np.array([500, 1000], np.int32), np.array([8.0, 12.0, 3.0]), ctx=ctx)
    assert list(got["clock_index"]) == [1, 0, -1]
    assert list(got["status"]) == [0, 0, 1]


# ---- full-size properties ------------------------------------------------------

def test_c2_full_size_properties(ctx):
    # BASELINE configs[1] at full size: 10k apps x 267 clocks, 500 trees depth 8.
    sc = W.make_scenario("c2", **W.CONFIGS["c2"])
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    first, e, t = gd.grid_select(me, mt, sc.grid, np.ones(sc.grid.n_apps), return_predictions=True)
    budgets = W.deadlines_from_times(t, seed=3)
    d1, e1, t1 = gd.grid_select(me, mt, sc.grid, budgets, return_predictions=True)
    d2 = gd.grid_select(me, mt, sc.grid, budgets)
    assert decisions_equal(d1, d2)  # determinism
    assert np.array_equal(bits(e1), bits(e)) and np.array_equal(bits(t1), bits(t))
    # decisions are the selection of the returned tables (K3 consistency)
    assert decisions_equal(O.oracle_select(e1, t1, sc.grid.sm, budgets), d1)
    # a seeded sample of apps against the oracle end to end
    idx = np.random.default_rng(0).choice(sc.grid.n_apps, 24, replace=False)
    sub = W.GridInputs(sc.grid.rows[idx], sc.grid.cat_t[idx], sc.grid.cat_cols, sc.grid.sm, sc.grid.mem, W.SM_COL,
                       W.MEM_COL)
    want, we, wt = O.oracle_grid(sc.energy, sc.time, sub, budgets[idx])
    assert np.array_equal(bits(e1[idx]), bits(we)) and np.array_equal(bits(t1[idx]), bits(wt))
    assert decisions_equal(d1[idx], want)
    # feasibility soundness (SPEC invariant): scheduled => T <= budget
    ok = (d1["status"] == 0) & (d1["note"] == 0)
    assert np.all(d1["time_s"][ok] <= budgets[ok])
    assert 0 < ok.sum() < sc.grid.n_apps


@pytest.mark.parametrize("wide", ["2", "0"])
@pytest.mark.parametrize("shape", ["c3", "c4"])
def test_deep_config_shapes_sampled_vs_oracle(ctx, shape, wide, monkeypatch):
    # BASELINE configs[2] / configs[3] at their full tree shapes (1000 trees
    # depth 10 on the 200-clock B200 grid; 2000 trees depth 12 on the
    # 267-clock grid), on slices of the very batches bench.py times (the same
    # chunk-seeded rows: apps [lo, hi) of the 1M / 10M-app batch).  128 apps
    # bit for bit against the REFERENCE's own predict + select (oracle/_ref,
    # all host threads) -- or 16 against the C oracle where _ref is absent --
    # and every app through the properties.  wide=2: the 1024-app walk tiles
    # with 8-bit ranks the bench's batches take; 0: 512-app tiles, 16-bit.
    monkeypatch.setenv("GDVFS_WIDE", wide)
    cfg = W.CONFIGS[shape]
    lo = 7 * W.CHUNK_APPS + 123  # inside the batch, across a chunk boundary
    n = 2048 if shape == "c3" else 1024
    sc = W.make_scenario("bench", cfg["n_apps"], cfg["catalog"], cfg["n_trees"], cfg["depth"], seed=1234,
                         chunked=True, app_range=(lo, lo + n))
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    _, e, t = gd.grid_select(me, mt, sc.grid, np.ones(sc.grid.n_apps), return_predictions=True)
    budgets = W.deadlines_from_times(t, seed=6)
    d1, e1, t1 = gd.grid_select(me, mt, sc.grid, budgets, return_predictions=True)
    assert np.array_equal(bits(e1), bits(e)) and np.array_equal(bits(t1), bits(t))
    assert decisions_equal(O.oracle_select(e1, t1, sc.grid.sm, budgets), d1)
    sample = 128 if O.ref_available() else 16
    idx = np.sort(np.random.default_rng(1).choice(sc.grid.n_apps, sample, replace=False))
    sub = W.GridInputs(sc.grid.rows[idx], sc.grid.cat_t[idx], sc.grid.cat_cols, sc.grid.sm, sc.grid.mem, W.SM_COL,
                       W.MEM_COL)
    if O.ref_available():
        _, want, we, wt = O.ref_bench_grid(sc.energy, sc.time, sub, budgets[idx], sample, os.cpu_count() or 1, tables=True)
    else:
        want, we, wt = O.oracle_grid(sc.energy, sc.time, sub, budgets[idx])
    assert np.array_equal(bits(e1[idx]), bits(we)) and np.array_equal(bits(t1[idx]), bits(wt))
    assert decisions_equal(d1[idx], want)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_c2_every_app_vs_reference(ctx):
    # BASELINE configs[1] at full size, EVERY one of the 10k apps against the
    # reference's own models::predict + schedule_d_dvfs (oracle/_ref, all
    # host threads): E/T tables and decisions bit for bit.
    sc = W.make_scenario("c2", **W.CONFIGS["c2"])
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    _, _, t = gd.grid_select(me, mt, sc.grid, np.ones(sc.grid.n_apps), return_predictions=True)
    budgets = W.deadlines_from_times(t, seed=3)
    got, ge, gt = gd.grid_select(me, mt, sc.grid, budgets, return_predictions=True)
    _, want, we, wt = O.ref_bench_grid(sc.energy, sc.time, sc.grid, budgets, sc.grid.n_apps, os.cpu_count() or 1,
                                              tables=True)
    assert np.array_equal(bits(ge), bits(we)) and np.array_equal(bits(gt), bits(wt))
    assert decisions_equal(got, want)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_trained_models_fast_path_vs_reference(ctx):
    # Ensembles TRAINED with the GPU fit_gbt on profiled records (clock
    # splits where the targets depend on the clocks, near the roots) through
    # the partial-evaluation path, against the reference's predict + select.
    sc = W.make_trained_scenario("trained", 600, "gtx980", 120, 8, seed=5, train_apps=24, stride=5, ctx=ctx)
    kinds = W.record_kinds(sc.time, sc.grid.rows, sc.grid.sm_col, sc.grid.mem_col, max_apps=16)
    assert kinds["CONST"] < 0.95  # the clock columns do matter to these models
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    _, _, t = gd.grid_select(me, mt, sc.grid, np.ones(sc.grid.n_apps), return_predictions=True)
    budgets = W.deadlines_from_times(t, seed=8)
    for opts in (gd.SchedulerOptions(budget="full"), gd.SchedulerOptions(budget="full", objective="power")):
        got, ge, gt = gd.grid_select(me, mt, sc.grid, budgets, opts, return_predictions=True)
        _, want, we, wt = O.ref_bench_grid(sc.energy, sc.time, sc.grid, budgets, sc.grid.n_apps, os.cpu_count() or 1,
                                              tables=True)
        assert np.array_equal(bits(ge), bits(we)) and np.array_equal(bits(gt), bits(wt))
        if opts.objective == "energy":
            assert decisions_equal(got, want)
        else:
            assert decisions_equal(got, O.oracle_select(we, wt, sc.grid.sm, budgets, objective=1))


def test_sum_tolerance_statement():
    # The kernels are bit-exact; north_star's 1e-5 relative tolerance is the
    # documented ceiling and is implied by 0-ulp equality above.
    assert REL_TOL == 1e-5


# ---- shapes outside the partial-evaluation pipeline: general kernel / chunked catalogs ----

def _check_vs_oracle(ctx, sc, grid=None, combos=((0, 0, 0), (1, 1, 1))):
    grid = grid or sc.grid
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    _, _, t0 = O.oracle_grid(sc.energy, sc.time, grid, np.ones(grid.n_apps))
    budgets = W.deadlines_from_times(t0, seed=4)
    for mode, obj, be in combos:
        opts = gd.SchedulerOptions(mode=["text", "literal"][mode], budget="full", objective=["energy", "power"][obj],
                                   best_effort_fallback=bool(be))
        want, we, wt = O.oracle_grid(sc.energy, sc.time, grid, budgets, mode, obj, be)
        got, ge, gt = gd.grid_select(me, mt, grid, budgets, opts, return_predictions=True)
        assert np.array_equal(bits(ge), bits(we)) and np.array_equal(bits(gt), bits(wt))
        assert decisions_equal(got, want)
        only = gd.grid_select(me, mt, grid, budgets, opts)
        assert decisions_equal(only, want)


@pytest.mark.parametrize("general", [False, True])
def test_wide_catalog_600_clocks(ctx, general):
    pairs = [(300 + 10 * i, m) for m in (405, 810, 2600, 3505, 5000, 6000) for i in range(100)]
    sm, mem = W._sorted_catalog(pairs)
    assert sm.shape[0] == 600
    sc = W.make_scenario("wide", 40, (sm, mem), 30, 6, seed=8, w_clk=0.2)
    grid = sc.grid
    if general:
        rng = np.random.default_rng(3)
        grid = W.GridInputs(grid.rows, grid.cat_t, grid.cat_cols, grid.sm, grid.mem, grid.sm_col, grid.mem_col,
                            rec_of_clock=rng.integers(0, 40, size=(40, 600)).astype(np.int32))
    _check_vs_oracle(ctx, sc, grid)
    # K3 alone over the same wide tables
    _, e, t = O.oracle_grid(sc.energy, sc.time, grid, np.full(40, 5.0))
    for mode in ("text", "literal"):
        opts = gd.SchedulerOptions(mode=mode, budget="full", best_effort_fallback=True)
        got = gd.select(e, t, grid.sm, np.full(40, 5.0), opts, ctx=ctx)
        want = O.oracle_select(e, t, grid.sm, np.full(40, 5.0), mode=int(mode == "literal"), best_effort=1)
        assert decisions_equal(got, want)


def test_clocks_above_16_bits_take_general_kernel(ctx):
    sm, mem = W._sorted_catalog([(70000 + 500 * i, 90000) for i in range(20)] + [(1000 + 10 * i, 405) for i in range(8)])
    sc = W.make_scenario("ghz", 50, (sm, mem), 25, 6, seed=2, w_clk=0.3)
    _check_vs_oracle(ctx, sc)


def test_many_thresholds_and_huge_trees_take_general_kernel(ctx):
    # > 65535 distinct thresholds on one feature (no 16-bit ranks) ...
    sc = W.make_scenario("thr", 30, "gtx980", 300, 8, seed=6, w_clk=0.05)
    rng = np.random.default_rng(0)
    for f in (sc.energy, sc.time):
        internal = (f.feature >= 0) & (f.feature != W.SM_COL) & (f.feature != W.MEM_COL)
        f.feature[internal] = 7
        f.threshold[internal] = sc.grid.rows[:, 7].mean() * np.exp(rng.uniform(-1, 1, int(internal.sum())))
    assert np.unique(sc.energy.threshold[sc.energy.feature == 7]).shape[0] > 65535
    _check_vs_oracle(ctx, sc)
    # ... and a tree of more than 65536 nodes (depth 16)
    big = W.make_scenario("big", 12, "p100", 2, 16, seed=3, w_clk=0.05)
    assert big.energy.n_nodes // 2 > 65536
    _check_vs_oracle(ctx, big, combos=((0, 0, 0),))


@pytest.mark.parametrize("stream", ["1", "0"])
def test_streamed_batch_inputs_vs_oracle(ctx, stream, monkeypatch):
    # A large host-buffer call of many app batches: rows / cat_t / budgets
    # are uploaded batch by batch on the copy stream while earlier batches
    # compute (GDVFS_STREAM_INPUTS=1), or in one upload first (0).
    monkeypatch.setenv("GDVFS_STREAM_INPUTS", stream)
    monkeypatch.setenv("GDVFS_BATCH_BYTES", "4000000")
    sc = W.make_scenario("streamed", 6000, "gtx980", 60, 8, seed=31, w_clk=0.08)
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    _, _, t0 = O.oracle_grid(sc.energy, sc.time, sc.grid, np.ones(sc.grid.n_apps))
    budgets = W.deadlines_from_times(t0, seed=4)
    want, we, wt = O.oracle_grid(sc.energy, sc.time, sc.grid, budgets)
    got = gd.grid_select(me, mt, sc.grid, budgets)
    assert decisions_equal(got, want)
    got2, ge, gt = gd.grid_select(me, mt, sc.grid, budgets, return_predictions=True)
    assert np.array_equal(bits(ge), bits(we)) and np.array_equal(bits(gt), bits(wt))
    assert decisions_equal(got2, want)


@pytest.mark.parametrize("fold", ["1", "0"])
def test_constant_clock_columns_folded_vs_oracle(ctx, fold, monkeypatch):
    # Catalogs whose memory (or core) clock is one value for every candidate:
    # those tests are folded into the walk nodes (GDVFS_FOLD=1) instead of
    # residues.  Catalogs alternate through the same models -- small calls
    # (staged, CUDA-graph replay) and large ones -- so folded walk nodes are
    # rebuilt, and stale graphs dropped, whenever the constancy changes.
    monkeypatch.setenv("GDVFS_FOLD", fold)
    sc = W.make_scenario("fold", 400, "gtx980", 60, 9, seed=41, w_clk=0.2)
    me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
    g = sc.grid
    sm_all, mem_all = g.sm.astype(np.int32), g.mem.astype(np.int32)
    one_mem = sm_all[mem_all == 3505]
    cats = {
        "single_mem": (one_mem, np.full(one_mem.shape, 3505, np.int32)),
        "single_sm": (np.full(4, 1185, np.int32), np.array([405, 810, 2600, 3505], np.int32)),
        "mixed": (sm_all, mem_all),
        "single_mem_other": (one_mem, np.full(one_mem.shape, 810, np.int32)),
    }
    for rep in range(2):
        for name, (sm, mem) in cats.items():
            for n in (64, 400):
                grid = W.GridInputs(g.rows[:n], g.cat_t[:n], g.cat_cols, sm, mem, g.sm_col, g.mem_col)
                _, _, t0 = O.oracle_grid(sc.energy, sc.time, grid, np.ones(n))
                budgets = W.deadlines_from_times(t0, seed=rep + 3)
                want, we, wt = O.oracle_grid(sc.energy, sc.time, grid, budgets)
                assert decisions_equal(gd.grid_select(me, mt, grid, budgets), want), (name, n, rep)
                got, ge, gt = gd.grid_select(me, mt, grid, budgets, return_predictions=True)
                assert np.array_equal(bits(ge), bits(we)) and np.array_equal(bits(gt), bits(wt)), (name, n, rep)
                assert decisions_equal(got, want), (name, n, rep)
                # the device-buffer path decides the folding on the device
                dt = _device_grid_select(ctx, me, mt, grid, budgets)
                assert np.array_equal(bits(dt), bits(wt)), (name, n, rep, "device path")


def _device_grid_select(ctx, me, mt, grid, budgets):
    """gd_grid_select_device on torch-resident copies of `grid`; returns the time table."""
    import torch

    dev = torch.device("cuda", 0)
    n, C_ = grid.rows.shape[0], len(grid.sm)
    keep = dict(rows=torch.from_numpy(np.ascontiguousarray(grid.rows)).to(dev),
                cat_t=torch.from_numpy(np.ascontiguousarray(grid.cat_t)).to(dev),
                cat_cols=torch.from_numpy(np.ascontiguousarray(grid.cat_cols, dtype=np.int32)).to(dev),
                sm=torch.from_numpy(np.ascontiguousarray(grid.sm, dtype=np.int32)).to(dev),
                mem=torch.from_numpy(np.ascontiguousarray(grid.mem, dtype=np.int32)).to(dev),
                budgets=torch.from_numpy(np.ascontiguousarray(budgets)).to(dev),
                out=torch.zeros(n * 24, dtype=torch.uint8, device=dev))
    t_tab = torch.empty((n, C_), dtype=torch.float64, device=dev)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    try:
        gd.grid_select_device(me, mt, {k: v.data_ptr() for k, v in keep.items()}, n, C_, grid.rows.shape[1],
                              grid.cat_t.shape[1], grid.sm_col, grid.mem_col, t_out=t_tab.data_ptr())
        torch.cuda.synchronize(dev)
    finally:
        ctx.set_stream(0)
    return t_tab.cpu().numpy()


@pytest.mark.parametrize("extra_cols", [70, 150])
def test_wide_rows_walk_geometry_fallbacks(ctx, extra_cols, monkeypatch):
    # Rows with many columns: the 8-bit 1024-app tile (F x 1024 B of ranks)
    # or even the 512-app one no longer leaves room for a tree pair, and the
    # walk geometry falls back to narrower tiles / fewer groups.  Streamed
    # batches and no categorical columns on the way.
    import dataclasses

    monkeypatch.setenv("GDVFS_BATCH_BYTES", "6000000")
    monkeypatch.setenv("GDVFS_WIDE", "2")
    sc = W.make_scenario("wide_rows", 3000, "gtx980", 50, 9, seed=17, w_clk=0.1)
    F = sc.grid.rows.shape[1] + extra_cols
    rows = np.concatenate([sc.grid.rows, np.random.default_rng(1).uniform(size=(3000, extra_cols))], axis=1)
    fe = dataclasses.replace(sc.energy, n_cols=F)
    ft = dataclasses.replace(sc.time, n_cols=F)
    grid = W.GridInputs(np.ascontiguousarray(rows), np.zeros((3000, 0)), np.zeros(0, np.int32), sc.grid.sm,
                        sc.grid.mem, sc.grid.sm_col, sc.grid.mem_col)
    me, mt = gd.Model.from_forest(fe, ctx), gd.Model.from_forest(ft, ctx)
    _, _, t0 = O.oracle_grid(fe, ft, grid, np.ones(3000))
    budgets = W.deadlines_from_times(t0, seed=2)
    want, we, wt = O.oracle_grid(fe, ft, grid, budgets)
    got, ge, gt = gd.grid_select(me, mt, grid, budgets, return_predictions=True)
    assert np.array_equal(bits(ge), bits(we)) and np.array_equal(bits(gt), bits(wt))
    assert decisions_equal(got, want)
