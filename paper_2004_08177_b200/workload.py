"""Seeded synthetic inputs for the (app x clock) evaluation path.

Everything here is deterministic in its seed and shared by the parity tests,
``bench.py`` and ``__graft_entry__.smoke()``, so the GPU path and the CPU
reference always consume identical bytes.

* Clock catalogs in ``clock_catalog`` order (mem asc, sm asc;
  reference core.cpp:177-184): the P100 62-clock grid
  (synthdata.cpp:271-287), the GTX-980-style 267-pair grid
  (tests/test_core.cpp:96-108) and a B200-style 200-clock grid.
* Ensembles in the reference's ``GbtTree`` node format (models.hpp:35-43):
  ``feature`` (-1 = leaf), ``threshold``, tree-local ``left``/``right``,
  ``leaf_value``, nodes in preorder as ``load_model`` produces them
  (models.cpp:581-607).  Thresholds are midpoints of two adjacent sorted pool
  values, like the trainer's split points (models.cpp:281).
* App rows with the reference's 50-column schema positions: categorical
  columns 0 (``double_precision_fu_utilisation``) and 3
  (``dram_utilisation``), ``mem_clock`` at 25 and ``sm_clock`` at 42
  (names sorted per ingest.cpp:21-34).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

N_COLS = 50
CAT_COLS = (0, 3)
MEM_COL = 25
SM_COL = 42


def _lround(x: float) -> int:
    """std::lround for the non-negative values used here (half away from zero)."""
    return int(math.floor(x + 0.5))


def _sorted_catalog(pairs):
    pairs = sorted(set(pairs), key=lambda p: (p[1], p[0]))
    sm = np.array([p[0] for p in pairs], dtype=np.int32)
    mem = np.array([p[1] for p in pairs], dtype=np.int32)
    return sm, mem


def catalog_p100():
    """synthdata.cpp:271-287: 62 sm clocks in [544, 1328] at mem 715, i=50 forced to 1189."""
    pairs = []
    for i in range(62):
        sm = _lround(544.0 + (1328.0 - 544.0) * i / 61.0)
        if i == 50:
            sm = 1189
        pairs.append((sm, 715))
    return _sorted_catalog(pairs)


def catalog_gtx980():
    """tests/test_core.cpp:96-108: mem {3505, 2600, 810} x 87 sm clocks + mem 405 x 6 = 267."""
    pairs = [(135 + 15 * i, mem) for mem in (3505, 2600, 810) for i in range(87)]
    pairs += [(135 + 15 * i, 405) for i in range(6)]
    return _sorted_catalog(pairs)


def catalog_b200(n: int = 200):
    """B200-style grid: mem 3996 MHz x n sm clocks lround-spaced over [510, 1965] MHz."""
    pairs = [(_lround(510.0 + (1965.0 - 510.0) * i / (n - 1)), 3996) for i in range(n)]
    return _sorted_catalog(pairs)


CATALOGS = {"p100": catalog_p100, "gtx980": catalog_gtx980, "b200": catalog_b200}


@dataclasses.dataclass
class Forest:
    """One GBT ensemble as flat SoA arrays (models::GbtParams + GbtTree nodes)."""

    tree_offsets: np.ndarray  # int64 [n_trees + 1]
    feature: np.ndarray  # int32, -1 = leaf
    threshold: np.ndarray  # float64
    left: np.ndarray  # int32, tree-local
    right: np.ndarray  # int32, tree-local
    leaf_value: np.ndarray  # float64
    base: float
    learning_rate: float
    target: int  # 0 energy (clamped at 0), 1 time
    n_cols: int

    @property
    def n_trees(self) -> int:
        return int(self.tree_offsets.shape[0] - 1)

    @property
    def n_nodes(self) -> int:
        return int(self.feature.shape[0])


@dataclasses.dataclass
class GridInputs:
    """Per-app rows (energy encoding) + time-encoded categorical values."""

    rows: np.ndarray  # float64 [n_records, n_cols]
    cat_t: np.ndarray  # float64 [n_records, n_cat]
    cat_cols: np.ndarray  # int32 [n_cat]
    sm: np.ndarray  # int32 [C]
    mem: np.ndarray  # int32 [C]
    sm_col: int
    mem_col: int
    rec_of_clock: Optional[np.ndarray] = None  # int32 [A, C] or None (record = app)

    @property
    def n_apps(self) -> int:
        if self.rec_of_clock is not None:
            return int(self.rec_of_clock.shape[0])
        return int(self.rows.shape[0])

    @property
    def n_clocks(self) -> int:
        return int(self.sm.shape[0])


def _preorder_perm(depth: int) -> np.ndarray:
    """Level-order index -> preorder index for a complete binary tree of `depth`."""
    n = (1 << (depth + 1)) - 1
    perm = np.empty(n, dtype=np.int64)
    counter = 0
    stack = [0]
    while stack:
        i = stack.pop()
        perm[i] = counter
        counter += 1
        l = 2 * i + 1
        if l < n:
            stack.append(l + 1)
            stack.append(l)
    return perm


class _ColumnModel:
    """Per-column value distributions (magnitudes 1e-2 .. 1e9, like the
    reference's counters) plus categorical level encodings per target."""

    def __init__(self, rng: np.random.Generator, n_cols: int, cat_cols, sm, mem, sm_col, mem_col):
        self.n_cols = n_cols
        self.cat_cols = tuple(cat_cols)
        self.sm_col, self.mem_col = sm_col, mem_col
        self.scale = 10.0 ** rng.uniform(-2.0, 9.0, size=n_cols)
        # four levels (none/low/mid/high) -> encoded values per target
        self.levels_e = np.sort(rng.uniform(20.0, 400.0, size=(len(self.cat_cols), 4)), axis=1)
        self.levels_t = np.sort(rng.uniform(0.5, 12.0, size=(len(self.cat_cols), 4)), axis=1)
        self.sm_vals = np.unique(sm).astype(np.float64)
        self.mem_vals = np.unique(mem).astype(np.float64)
        self.pool = self.scale[None, :] * np.exp(rng.uniform(-1.0, 1.0, size=(256, n_cols)))
        self.pool.sort(axis=0)

    def thresholds(self, rng: np.random.Generator, feat: np.ndarray, target: int) -> np.ndarray:
        thr = np.empty(feat.shape, dtype=np.float64)
        k = rng.integers(0, 255, size=feat.shape)
        thr[:] = 0.5 * (self.pool[k, feat] + self.pool[k + 1, feat])
        for ci, c in enumerate(self.cat_cols):
            m = feat == c
            lv = self.levels_e[ci] if target == 0 else self.levels_t[ci]
            j = rng.integers(0, 3, size=int(m.sum()))
            thr[m] = 0.5 * (lv[j] + lv[j + 1])
        for col, vals in ((self.sm_col, self.sm_vals), (self.mem_col, self.mem_vals)):
            m = feat == col
            if not m.any():
                continue
            if len(vals) < 2:
                thr[m] = vals[0] + 0.5
                continue
            j = rng.integers(0, len(vals) - 1, size=int(m.sum()))
            thr[m] = 0.5 * (vals[j] + vals[j + 1])
        return thr


def make_forest(cols: _ColumnModel, n_trees: int, depth: int, target: int, seed: int,
                w_clk: float = 0.04, leaf_prob: float = 0.0) -> Forest:
    """Random ensemble in reference node format.

    Complete trees of `depth` (preorder ids) when leaf_prob == 0; otherwise
    each internal node below the root turns into a leaf with probability
    `leaf_prob` (irregular trees, explicit children, still preorder).
    A fraction `w_clk` of split features are the clock columns.
    """
    rng = np.random.default_rng(seed)
    base = 180.0 if target == 0 else 6.0
    scale = 120.0 if target == 0 else 4.0
    non_clock = np.array([c for c in range(cols.n_cols) if c not in (cols.sm_col, cols.mem_col)])
    if leaf_prob <= 0.0:
        n_int = (1 << depth) - 1
        n = (1 << (depth + 1)) - 1
        perm = _preorder_perm(depth)
        feat_lv = non_clock[rng.integers(0, len(non_clock), size=(n_trees, n_int))]
        clk = rng.random(size=(n_trees, n_int)) < w_clk
        which = rng.random(size=(n_trees, n_int)) < 0.5
        feat_lv = np.where(clk, np.where(which, cols.sm_col, cols.mem_col), feat_lv).astype(np.int32)
        thr_lv = cols.thresholds(rng, feat_lv, target)
        leaf_lv = rng.uniform(-1.0, 1.0, size=(n_trees, n - n_int)) * scale
        feature = np.full((n_trees, n), -1, dtype=np.int32)
        threshold = np.zeros((n_trees, n), dtype=np.float64)
        left = np.full((n_trees, n), -1, dtype=np.int32)
        right = np.full((n_trees, n), -1, dtype=np.int32)
        leaf = np.zeros((n_trees, n), dtype=np.float64)
        lv = np.arange(n)
        pi = perm[lv[:n_int]]
        feature[:, pi] = feat_lv
        threshold[:, pi] = thr_lv
        left[:, pi] = perm[2 * lv[:n_int] + 1]
        right[:, pi] = perm[2 * lv[:n_int] + 2]
        leaf[:, perm[lv[n_int:]]] = leaf_lv
        offsets = np.arange(n_trees + 1, dtype=np.int64) * n
        return Forest(offsets, feature.ravel(), threshold.ravel(), left.ravel(), right.ravel(),
                      leaf.ravel(), base, 0.1, target, cols.n_cols)

    feats, thrs, lefts, rights, leaves, offsets = [], [], [], [], [], [0]
    for _ in range(n_trees):
        f_t, th_t, l_t, r_t, v_t = [], [], [], [], []

        def build(d):
            idx = len(f_t)
            f_t.append(-1); th_t.append(0.0); l_t.append(-1); r_t.append(-1); v_t.append(0.0)
            if d == depth or (d > 0 and rng.random() < leaf_prob):
                v_t[idx] = float(rng.uniform(-1.0, 1.0) * scale)
                return idx
            if rng.random() < w_clk:
                f = cols.sm_col if rng.random() < 0.5 else cols.mem_col
            else:
                f = int(non_clock[rng.integers(0, len(non_clock))])
            f_t[idx] = f
            th_t[idx] = float(cols.thresholds(rng, np.array([f]), target)[0])
            l_t[idx] = build(d + 1)
            r_t[idx] = build(d + 1)
            return idx

        build(0)
        feats += f_t; thrs += th_t; lefts += l_t; rights += r_t; leaves += v_t
        offsets.append(offsets[-1] + len(f_t))
    return Forest(np.array(offsets, dtype=np.int64), np.array(feats, dtype=np.int32),
                  np.array(thrs, dtype=np.float64), np.array(lefts, dtype=np.int32),
                  np.array(rights, dtype=np.int32), np.array(leaves, dtype=np.float64),
                  base, 0.1, target, cols.n_cols)


def make_rows(cols: _ColumnModel, n_apps: int, seed: int, sm_default: int, mem_default: int):
    rng = np.random.default_rng(seed)
    rows = cols.scale[None, :] * np.exp(rng.uniform(-1.0, 1.0, size=(n_apps, cols.n_cols)))
    cat_t = np.empty((n_apps, len(cols.cat_cols)), dtype=np.float64)
    for ci, c in enumerate(cols.cat_cols):
        lvl = rng.integers(0, 4, size=n_apps)
        rows[:, c] = cols.levels_e[ci][lvl]
        cat_t[:, ci] = cols.levels_t[ci][lvl]
    rows[:, cols.sm_col] = float(sm_default)
    rows[:, cols.mem_col] = float(mem_default)
    return np.ascontiguousarray(rows), np.ascontiguousarray(cat_t)


CHUNK_APPS = 1 << 16  # apps per independently seeded chunk (large configs)


def _rows_chunk(cols: _ColumnModel, seed: int, chunk: int, sm_default: int, mem_default: int):
    return make_rows(cols, CHUNK_APPS, hash_seed(seed, 0x524f5753, chunk), sm_default, mem_default)


def make_rows_range(cols: _ColumnModel, lo: int, hi: int, seed: int, sm_default: int, mem_default: int,
                    threads: int = 0):
    """Rows of apps [lo, hi) of a chunk-seeded scenario: chunk k (apps
    [k*CHUNK_APPS, (k+1)*CHUNK_APPS)) draws from its own seed, so any app
    range -- one rank's shard of configs[3]'s 10M apps, or the reference
    arm's sample -- is generated alone and matches the whole batch's rows."""
    n = hi - lo
    rows = np.empty((n, cols.n_cols), np.float64)
    cat_t = np.empty((n, len(cols.cat_cols)), np.float64)
    if n <= 0:
        return rows, cat_t
    k0, k1 = lo // CHUNK_APPS, (hi - 1) // CHUNK_APPS

    def one(k):
        r, c = _rows_chunk(cols, seed, k, sm_default, mem_default)
        a, b = max(lo, k * CHUNK_APPS), min(hi, (k + 1) * CHUNK_APPS)
        rows[a - lo:b - lo] = r[a - k * CHUNK_APPS:b - k * CHUNK_APPS]
        cat_t[a - lo:b - lo] = c[a - k * CHUNK_APPS:b - k * CHUNK_APPS]

    ks = range(k0, k1 + 1)
    if threads != 1 and len(ks) > 1:
        from concurrent.futures import ThreadPoolExecutor
        import os
        with ThreadPoolExecutor(threads or min(16, os.cpu_count() or 1)) as ex:
            list(ex.map(one, ks))
    else:
        for k in ks:
            one(k)
    return rows, cat_t


def hash_seed(*parts: int) -> int:
    """SplitMix64 over the parts (a counter-based seed: chunk k of seed s is
    the same whatever else is generated)."""
    x = 0
    for p in parts:
        x = (x + 0x9E3779B97F4A7C15 + (int(p) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        x = z ^ (z >> 31)
    return x


@dataclasses.dataclass
class Scenario:
    name: str
    energy: Forest
    time: Forest
    grid: GridInputs
    seed: int
    cols: Optional[_ColumnModel] = None
    app_range: tuple = (0, 0)  # global indices of grid's apps (chunked scenarios)

    def rows_range(self, lo: int, hi: int):
        """Rows + time-encoded categorical values of global apps [lo, hi)
        (chunk-seeded scenarios only)."""
        sm, mem = self.grid.sm, self.grid.mem
        return make_rows_range(self.cols, lo, hi, self.seed + 3, int(sm[-1]), int(mem[-1]))


def make_scenario(name: str, n_apps: int, catalog, n_trees: int, depth: int, seed: int = 1234,
                  w_clk: float = 0.04, leaf_prob: float = 0.0, chunked: Optional[bool] = None,
                  app_range: Optional[tuple] = None) -> Scenario:
    """A complete synthetic (apps, catalog, E/T ensembles) configuration.
    `catalog`: a CATALOGS name or an explicit (sm, mem) pair of int32 arrays
    in the order the candidates are to be evaluated (any order).

    Batches above CHUNK_APPS apps (configs[2] / configs[3]) draw their rows
    chunk by chunk (`make_rows_range`); `app_range=(lo, hi)` then builds only
    those apps of the n_apps-app batch (one rank's shard, a CPU sample)."""
    if isinstance(catalog, str):
        sm, mem = CATALOGS[catalog]()
    else:
        sm, mem = (np.ascontiguousarray(x, dtype=np.int32) for x in catalog)
    rng = np.random.default_rng(seed)
    cols = _ColumnModel(rng, N_COLS, CAT_COLS, sm, mem, SM_COL, MEM_COL)
    fe = make_forest(cols, n_trees, depth, 0, seed + 1, w_clk, leaf_prob)
    ft = make_forest(cols, n_trees, depth, 1, seed + 2, w_clk, leaf_prob)
    if chunked is None:
        chunked = n_apps > CHUNK_APPS or app_range is not None
    lo, hi = app_range if app_range is not None else (0, n_apps)
    if chunked:
        rows, cat_t = make_rows_range(cols, lo, hi, seed + 3, int(sm[-1]), int(mem[-1]))
    else:
        rows, cat_t = make_rows(cols, n_apps, seed + 3, int(sm[-1]), int(mem[-1]))
    grid = GridInputs(rows, cat_t, np.array(CAT_COLS, dtype=np.int32), sm, mem, SM_COL, MEM_COL)
    return Scenario(name, fe, ft, grid, seed, cols, (lo, hi))


# ---- trained models -----------------------------------------------------------
#
# The synthetic ensembles above are random trees with a fixed clock-split
# rate.  The scenario below instead TRAINS both ensembles (fit_gbt on the GPU,
# the reference's exact booster) on profiled records of a roofline
# application model, the shape of the reference's synthetic GPU
# (synthdata.cpp: time = max(compute / sm, memory / mem) + stall, power from
# the utilisations, counters proportional to the work, throughputs = counter /
# time, a binned utilisation as a categorical column, clock-keyed
# distractors).  Trained trees split on the clock columns wherever the target
# depends on them -- near the root, with the distribution of clock residues a
# production model has.


def _archetypes(n: int, seed: int):
    r = np.random.default_rng(seed)
    return dict(cw=r.uniform(420.0, 5300.0, n), mw=r.uniform(70.0, 1950.0, n), stall=r.uniform(0.10, 1.40, n),
                kc=r.uniform(0.034, 0.105, n), km=r.uniform(0.007, 0.058, n), gain=r.uniform(0.7, 1.3, (n, 16)),
                key=r.integers(0, 2**31, n))


def _profiles(arch, idx, sm, mem):
    """Profiled rows (the 50-column schema), energy and time for app idx x
    clocks (sm, mem) (flat arrays of equal length)."""
    cw, mw, st = arch["cw"][idx], arch["mw"][idx], arch["stall"][idx]
    g = arch["gain"][idx]
    smf, memf = sm.astype(np.float64), mem.astype(np.float64)
    tc, tm = cw / smf, mw / memf
    t_det = np.maximum(tc, tm) + st
    uc, um = tc / t_det, tm / t_det
    stall_frac = st / t_det
    volt = 0.70 + 0.35 * (smf - 135.0) / 1800.0
    power = 30.0 + arch["kc"][idx] * smf * volt * volt * uc + arch["km"][idx] * memf * um
    rows = np.zeros((len(idx), N_COLS))
    counters = [cw * 250.0, cw * 620.0, cw * 45.0, cw * 110.0, cw * 55.0, mw * 31250.0, mw * 1.0e6, mw * 11000.0,
                mw * 48000.0, mw * 26000.0, mw * 8000.0 + cw * 900.0, mw * 7.3e5, (cw + mw) * 1800.0,
                (cw + mw) * 2600.0]
    free = [c for c in range(N_COLS) if c not in CAT_COLS and c not in (SM_COL, MEM_COL)]
    k = 0
    for j, c in enumerate(counters):
        rows[:, free[k]] = c * g[:, j % 16]
        k += 1
    for j, c in enumerate(counters[:8]):  # throughputs: counter / time
        rows[:, free[k]] = c * g[:, (j + 3) % 16] / t_det / 1e9
        k += 1
    for v in (100.0 * uc, 4.0 * uc * (1 - 0.6 * stall_frac), 100.0 * (1 - 0.55 * um), 100.0 * (0.55 + 0.45 * uc),
              100.0 * stall_frac * 0.55, 100.0 * np.minimum(1.0, 0.5 * um), 0.03 + 0.12 * um,
              8.0 * uc * (1 - 0.5 * stall_frac)):
        rows[:, free[k]] = v
        k += 1
    while k < len(free):  # distractors keyed by (app, clock)
        h = (arch["key"][idx] * 1000003 + sm * 7919 + mem * 104729 + k * 15485863) % 1000003
        rows[:, free[k]] = 100.0 * h / 1000003.0
        k += 1
    rows[:, SM_COL], rows[:, MEM_COL] = smf, memf
    lvl_u = np.minimum((um * 4).astype(int), 3)  # binned utilisations (categorical levels)
    lvl_c = np.minimum((uc * 4).astype(int), 3)
    time = t_det * (1.0 + 0.01 * np.sin(arch["key"][idx] + smf))
    energy = power * time
    return rows, (lvl_c, lvl_u), energy, time


def make_trained_scenario(name: str, n_apps: int, catalog, n_trees: int, depth: int, seed: int = 1234,
                          train_apps: int = 48, stride: int = 3, ctx=None,
                          app_range: Optional[tuple] = None) -> Scenario:
    """(apps, catalog, E/T ensembles TRAINED on profiled records with the
    GPU fit_gbt).  Training set: `train_apps` archetypes x every `stride`-th
    catalog clock; categorical levels encoded by their mean target per
    target (so the time model sees its own values, cat_t).  Query rows: the
    default-clock (max sm, max mem) profile of `n_apps` further archetypes."""
    import paper_2004_08177_b200 as gd

    if isinstance(catalog, str):
        sm, mem = CATALOGS[catalog]()
    else:
        sm, mem = (np.ascontiguousarray(x, dtype=np.int32) for x in catalog)
    lo, hi = app_range if app_range is not None else (0, n_apps)
    arch = _archetypes(train_apps + n_apps, seed)
    ci = np.arange(0, sm.shape[0], stride)
    ia = np.repeat(np.arange(train_apps), ci.shape[0])
    ic = np.tile(ci, train_apps)
    rows, (lc, lu), energy, time = _profiles(arch, ia, sm[ic], mem[ic])
    enc = {}
    for tgt, y in ((0, energy), (1, time)):
        vals = []
        for lv in (lc, lu):
            m = np.array([y[lv == k].mean() if np.any(lv == k) else y.mean() for k in range(4)])
            vals.append(m)
        enc[tgt] = vals
    def encode(r, lvls, tgt):
        out = r.copy()
        for ci_, (c, lv) in enumerate(zip(CAT_COLS, lvls)):
            out[:, c] = enc[tgt][ci_][lv]
        return out
    xe, xt = encode(rows, (lc, lu), 0), encode(rows, (lc, lu), 1)
    me = gd.fit_gbt(xe, energy, n_trees, depth, 0.1, 3.0, seed, 0, ctx=ctx)
    mt = gd.fit_gbt(xt, time, n_trees, depth, 0.1, 3.0, seed, 1, ctx=ctx)
    fe, ft = me.export(), mt.export()
    me.close()
    mt.close()
    qa = np.arange(train_apps + lo, train_apps + hi)
    d_sm, d_mem = np.full(hi - lo, int(sm.max()), np.int32), np.full(hi - lo, int(mem.max()), np.int32)
    qrows, (qc, qu), _, _ = _profiles(arch, qa, d_sm, d_mem)
    q_e = encode(qrows, (qc, qu), 0)
    q_t = encode(qrows, (qc, qu), 1)
    cat_t = np.ascontiguousarray(q_t[:, list(CAT_COLS)])
    grid = GridInputs(np.ascontiguousarray(q_e), cat_t, np.array(CAT_COLS, dtype=np.int32), sm, mem, SM_COL, MEM_COL)
    return Scenario(name, fe, ft, grid, seed, None, (lo, hi))


def record_kinds(forest: Forest, rows: np.ndarray, sm_col: int, mem_col: int, max_apps: int = 64) -> dict:
    """Share of (app, tree) pairs per walk-record kind (what the walk kernel
    emits): CONST (row-only walk ends on a leaf), SM / MEM (one clock test
    between two leaves), TABLE (2-3 test levels), TABLE4 (4), FULL (deeper).
    CPU analysis over the first `max_apps` rows -- a measurement aid."""
    off, f, th, le, ri = forest.tree_offsets, forest.feature, forest.threshold, forest.left, forest.right

    def walk(o, n, row):
        while True:
            ft = f[o + n]
            if ft < 0 or ft == sm_col or ft == mem_col:
                return n
            n = le[o + n] if row[ft] <= th[o + n] else ri[o + n]

    def levels(o, n, row):  # test levels of the clock-only residue below node n
        n = walk(o, n, row)
        if f[o + n] < 0:
            return 0
        return 1 + max(levels(o, le[o + n], row), levels(o, ri[o + n], row))

    counts = dict(CONST=0, SM=0, MEM=0, TABLE=0, TABLE4=0, FULL=0)
    n_apps = min(max_apps, rows.shape[0])
    for a in range(n_apps):
        row = rows[a]
        for t in range(forest.n_trees):
            o = int(off[t])
            d = levels(o, 0, row)
            if d == 0:
                counts["CONST"] += 1
            elif d == 1:
                counts["SM" if f[o + walk(o, 0, row)] == sm_col else "MEM"] += 1
            elif d <= 3:
                counts["TABLE"] += 1
            elif d == 4:
                counts["TABLE4"] += 1
            else:
                counts["FULL"] += 1
    tot = max(1, n_apps * forest.n_trees)
    return {k: round(v / tot, 4) for k, v in counts.items()}


def deadlines_from_times(times: np.ndarray, seed: int, infeasible_frac: float = 0.05) -> np.ndarray:
    """Per-app relative deadline: a seeded quantile q ~ U(0.1, 0.9) of the app's own
    predicted times over the grid; `infeasible_frac` of apps
    get half their minimum time so the rejected / best-effort paths run."""
    rng = np.random.default_rng(seed)
    a = times.shape[0]
    q = rng.uniform(0.1, 0.9, size=a)
    srt = np.sort(times, axis=1)
    idx = np.minimum((q * (times.shape[1] - 1)).astype(np.int64), times.shape[1] - 1)
    dl = srt[np.arange(a), idx].copy()
    bad = rng.random(size=a) < infeasible_frac
    dl[bad] = srt[bad, 0] * 0.5
    return dl


def deadline_draws(seed: int, lo: int, hi: int, infeasible_frac: float = 0.05):
    """Per-app deadline draws of `deadlines_from_times` for global apps
    [lo, hi), chunk-seeded like the rows: the quantile q ~ U(0.1, 0.9) and the
    `bad` flag (deadline = half the minimum time) of app i are the same in
    any app range, so the reference arm's sample and every rank's shard see
    the deadlines of the whole batch."""
    n = max(hi - lo, 0)
    q = np.empty(n)
    bad = np.empty(n, bool)
    if n == 0:
        return q, bad
    for k in range(lo // CHUNK_APPS, (hi - 1) // CHUNK_APPS + 1):
        r = np.random.default_rng(hash_seed(seed, 0x444c, k))
        qk = r.uniform(0.1, 0.9, size=CHUNK_APPS)
        bk = r.random(size=CHUNK_APPS) < infeasible_frac
        a, b = max(lo, k * CHUNK_APPS), min(hi, (k + 1) * CHUNK_APPS)
        q[a - lo:b - lo] = qk[a - k * CHUNK_APPS:b - k * CHUNK_APPS]
        bad[a - lo:b - lo] = bk[a - k * CHUNK_APPS:b - k * CHUNK_APPS]
    return q, bad


def deadlines_from_draws(times: np.ndarray, q: np.ndarray, bad: np.ndarray) -> np.ndarray:
    """The deadlines_from_times rule for given draws (numpy; bench.py runs the
    same rule on device tensors)."""
    srt = np.sort(times, axis=1)
    c = times.shape[1]
    idx = np.minimum((q * (c - 1)).astype(np.int64), c - 1)
    dl = srt[np.arange(times.shape[0]), idx].copy()
    dl[bad] = srt[bad, 0] * 0.5
    return dl


# The BASELINE.json configurations.
CONFIGS = {
    "c2": dict(n_apps=10_000, catalog="gtx980", n_trees=500, depth=8),
    "c3": dict(n_apps=1_000_000, catalog="b200", n_trees=1000, depth=10),
    "c4": dict(n_apps=10_000_000, catalog="gtx980", n_trees=2000, depth=12),
    "c5": dict(n_apps=64, catalog="gtx980", n_trees=500, depth=8),
    # configs[1] shape with ensembles TRAINED on profiled records (GPU fit_gbt)
    "c2t": dict(n_apps=10_000, catalog="gtx980", n_trees=500, depth=8, trained=True),
}
