"""ctypes bindings for the CHECKERS: oracle/liboracle.so (C restatement) and
oracle/_ref/libgpudvfs_ref.so (the reference's own sources compiled).

Test infrastructure only -- imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg, never by the product package.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path
from typing import Optional

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
ORACLE_SO = ORACLE_DIR / "liboracle.so"
REF_SO = ORACLE_DIR / "_ref" / "libgpudvfs_ref.so"
REF_SRC = Path("/root/reference/proj")

DECISION_DTYPE = np.dtype([("clock_index", "<i4"), ("status", "<i2"), ("note", "<i2"), ("energy_ws", "<f8"),
                           ("time_s", "<f8")])
assert DECISION_DTYPE.itemsize == 24
JOB_DTYPE = np.dtype([("arrival_s", "<f8"), ("deadline_s", "<f8"), ("app_rank", "<i8"), ("app_index", "<i4"),
                      ("pad", "<i4")])


class ForestView(C.Structure):
    _fields_ = [("n_trees", C.c_int32), ("tree_offsets", C.c_void_p), ("feature", C.c_void_p),
                ("threshold", C.c_void_p), ("left", C.c_void_p), ("right", C.c_void_p),
                ("leaf_value", C.c_void_p)]


def _p(a):
    return None if a is None else a.ctypes.data


def forest_view(f):
    keep = [np.ascontiguousarray(f.tree_offsets, np.int64), np.ascontiguousarray(f.feature, np.int32),
            np.ascontiguousarray(f.threshold, np.float64), np.ascontiguousarray(f.left, np.int32),
            np.ascontiguousarray(f.right, np.int32), np.ascontiguousarray(f.leaf_value, np.float64)]
    return ForestView(f.n_trees, *[k.ctypes.data for k in keep]), keep


def build_oracle(ref: bool = True) -> None:
    """Compile the checkers (oracle/Makefile); _ref only where the reference exists."""
    targets = ["oracle"] + (["ref"] if ref and REF_SRC.exists() else [])
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "-j8", *targets], check=True)


_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not ORACLE_SO.exists():
            build_oracle(ref=False)
        o = C.CDLL(str(ORACLE_SO))
        P = C.c_void_p
        o.gdo_leaf_index.restype = C.c_int32
        o.gdo_leaf_index.argtypes = [C.POINTER(ForestView), C.c_int32, P]
        o.gdo_predict_gbt.argtypes = [C.POINTER(ForestView), C.c_double, C.c_double, C.c_int32, P, C.c_int64,
                                      C.c_int32, P, P]
        o.gdo_predict_linear.argtypes = [P, C.c_double, C.c_int32, P, C.c_int64, C.c_int32, P]
        o.gdo_select.argtypes = [P, P, P, C.c_int32, C.c_double, C.c_int32, C.c_int32, C.c_int32, P]
        o.gdo_grid_select.argtypes = [C.POINTER(ForestView), C.c_double, C.c_double, C.POINTER(ForestView),
                                      C.c_double, C.c_double, P, C.c_int64, C.c_int32, P, P, C.c_int32, P,
                                      C.c_int64, P, P, C.c_int32, C.c_int32, C.c_int32, P, C.c_int32, C.c_int32,
                                      C.c_int32, P, P, P]
        o.gdo_schedule_edf.argtypes = [P, C.c_int64, P, P, P, P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.c_int32, P, P]
        _oracle = o
    return _oracle


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> Optional[C.CDLL]:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            return None
        r = C.CDLL(str(REF_SO))
        P = C.c_void_p
        r.ref_last_error.restype = C.c_char_p
        r.ref_predict_forest.argtypes = [C.POINTER(ForestView), C.c_double, C.c_double, C.c_int, P, C.c_int64,
                                         C.c_int, P]
        r.ref_save_forest.argtypes = [C.POINTER(ForestView), C.c_double, C.c_double, C.c_int, C.c_int, C.c_char_p]
        r.ref_predict_model_file.argtypes = [C.c_char_p, P, C.c_int64, C.c_int, P]
        r.ref_predict_column_mismatch.argtypes = [C.c_char_p, P, C.c_int, C.c_char_p, C.c_int]
        r.ref_schedule_tables.argtypes = [P, C.c_int64, P, P, P, P, P, C.c_int32, C.c_int, C.c_int, C.c_int,
                                          C.c_int, P, P]
        r.ref_c1_scenario.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.c_int, C.c_int, C.c_int]
        r.ref_truth_oracle.argtypes = [C.c_uint64, P, P, P, P, P]
        r.ref_c1_train.argtypes = [C.c_uint64, C.c_int, C.c_int, P, P, P, P]
        r.ref_fit_gbt.argtypes = [P, C.c_int64, C.c_int, P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                  C.c_int, P, P, P]
        r.ref_fit_gbt_export.argtypes = [P, P, P, P, P, P]
        r.ref_bench_grid.restype = C.c_double
        r.ref_bench_grid.argtypes = [C.POINTER(ForestView), C.c_double, C.c_double, C.POINTER(ForestView),
                                     C.c_double, C.c_double, P, C.c_int, P, P, C.c_int, C.c_int64, P, P, C.c_int32,
                                     C.c_int, C.c_int, P, C.c_int, P, P, P]
        _ref = r
    return _ref


def _ref_check(rc):
    if rc != 0:
        raise RuntimeError(ref().ref_last_error().decode())


# ---- oracle wrappers --------------------------------------------------------

def oracle_predict(forest, rows, leaf_ids=False):
    rows = np.ascontiguousarray(rows, np.float64)
    fv, keep = forest_view(forest)
    out = np.empty(rows.shape[0], np.float64)
    ids = np.empty((rows.shape[0], forest.n_trees), np.int32) if leaf_ids else None
    oracle().gdo_predict_gbt(C.byref(fv), forest.base, forest.learning_rate, int(forest.target == 0), _p(rows),
                             rows.shape[0], rows.shape[1], _p(out), _p(ids))
    return (out, ids) if leaf_ids else out


def oracle_predict_linear(coef, intercept, clamp, rows):
    rows = np.ascontiguousarray(rows, np.float64)
    coef = np.ascontiguousarray(coef, np.float64)
    out = np.empty(rows.shape[0], np.float64)
    oracle().gdo_predict_linear(_p(coef), intercept, clamp, _p(rows), rows.shape[0], rows.shape[1], _p(out))
    return out


def oracle_select(E, T, sm, budgets, mode=0, objective=0, best_effort=0):
    E = np.ascontiguousarray(E, np.float64)
    T = np.ascontiguousarray(T, np.float64)
    sm = np.ascontiguousarray(sm, np.int32)
    out = np.zeros(E.shape[0], DECISION_DTYPE)
    one = np.zeros(1, DECISION_DTYPE)
    for a in range(E.shape[0]):
        oracle().gdo_select(_p(E[a]), _p(T[a]), _p(sm), E.shape[1], float(budgets[a]), mode, objective,
                            best_effort, _p(one))
        out[a] = one[0]
    return out


def oracle_grid(fe, ft, grid, budgets, mode=0, objective=0, best_effort=0, app_slice=None):
    rows = np.ascontiguousarray(grid.rows, np.float64)
    cat_t = np.ascontiguousarray(grid.cat_t, np.float64)
    cat_cols = np.ascontiguousarray(grid.cat_cols, np.int32)
    rec = None if grid.rec_of_clock is None else np.ascontiguousarray(grid.rec_of_clock, np.int32)
    sm = np.ascontiguousarray(grid.sm, np.int32)
    mem = np.ascontiguousarray(grid.mem, np.int32)
    budgets = np.ascontiguousarray(budgets, np.float64)
    a0, a1 = (0, grid.n_apps) if app_slice is None else app_slice
    n = a1 - a0
    C_ = sm.shape[0]
    if rec is None:
        rows_v, cat_v, rec_v = rows[a0:a1], cat_t[a0:a1], None
    else:
        rows_v, cat_v, rec_v = rows, cat_t, np.ascontiguousarray(rec[a0:a1])
    out = np.zeros(n, DECISION_DTYPE)
    e = np.empty((n, C_), np.float64)
    t = np.empty((n, C_), np.float64)
    fve, k1 = forest_view(fe)
    fvt, k2 = forest_view(ft)
    oracle().gdo_grid_select(C.byref(fve), fe.base, fe.learning_rate, C.byref(fvt), ft.base, ft.learning_rate,
                             _p(np.ascontiguousarray(rows_v)), rows_v.shape[0], rows.shape[1],
                             _p(np.ascontiguousarray(cat_v)), _p(cat_cols), cat_cols.shape[0], _p(rec_v), n, _p(sm),
                             _p(mem), C_, grid.sm_col, grid.mem_col, _p(np.ascontiguousarray(budgets[a0:a1])), mode,
                             objective, best_effort, _p(out), _p(e), _p(t))
    return out, e, t


def oracle_schedule(jobs, E, T, exec_time, sm, mode=0, budget=0, objective=0, best_effort=0):
    jobs = np.ascontiguousarray(jobs, JOB_DTYPE)
    n = jobs.shape[0]
    out = np.zeros(n, DECISION_DTYPE)
    order = np.zeros(n, np.int64)
    E = np.ascontiguousarray(E, np.float64)
    T = np.ascontiguousarray(T, np.float64)
    X = np.ascontiguousarray(exec_time, np.float64)
    sm = np.ascontiguousarray(sm, np.int32)
    oracle().gdo_schedule_edf(_p(jobs), n, _p(E), _p(T), _p(X), _p(sm), sm.shape[0], mode, budget, objective,
                              best_effort, _p(out), _p(order))
    return out, order


# ---- reference wrappers ------------------------------------------------------

def ref_predict(forest, rows):
    rows = np.ascontiguousarray(rows, np.float64)
    fv, keep = forest_view(forest)
    out = np.empty(rows.shape[0], np.float64)
    _ref_check(ref().ref_predict_forest(C.byref(fv), forest.base, forest.learning_rate, forest.target, _p(rows),
                                        rows.shape[0], rows.shape[1], _p(out)))
    return out


def ref_c1_train(seed=7, stride=2, target=0):
    """The C1 catalog's encoded training matrix (rows, targets) from the reference."""
    n, p = C.c_int64(), C.c_int32()
    _ref_check(ref().ref_c1_train(seed, stride, target, None, None, C.byref(n), C.byref(p)))
    rows = np.empty((n.value, p.value), np.float64)
    targets = np.empty(n.value, np.float64)
    _ref_check(ref().ref_c1_train(seed, stride, target, _p(rows), _p(targets), C.byref(n), C.byref(p)))
    return rows, targets


def ref_fit_gbt(rows, targets, iterations, depth, lr=0.1, l2=3.0, seed=7, target=0):
    """models::fit_gbt on (rows, targets): the Forest in fit_gbt's own node order."""
    from paper_2004_08177_b200.workload import Forest

    rows = np.ascontiguousarray(rows, np.float64)
    targets = np.ascontiguousarray(targets, np.float64)
    nt, nn, base = C.c_int32(), C.c_int64(), C.c_double()
    _ref_check(ref().ref_fit_gbt(_p(rows), rows.shape[0], rows.shape[1], _p(targets), iterations, depth, lr, l2, seed,
                                 target, C.byref(nt), C.byref(nn), C.byref(base)))
    off = np.empty(nt.value + 1, np.int64)
    f, l, r = (np.empty(nn.value, np.int32) for _ in range(3))
    th, lv = np.empty(nn.value, np.float64), np.empty(nn.value, np.float64)
    _ref_check(ref().ref_fit_gbt_export(_p(off), _p(f), _p(th), _p(l), _p(r), _p(lv)))
    return Forest(off, f, th, l, r, lv, base.value, lr, target, rows.shape[1])


def ref_save_forest(forest, path):
    fv, keep = forest_view(forest)
    _ref_check(ref().ref_save_forest(C.byref(fv), forest.base, forest.learning_rate, forest.target, forest.n_cols,
                                     str(path).encode()))


def ref_predict_model_file(path, rows):
    rows = np.ascontiguousarray(rows, np.float64)
    out = np.empty(rows.shape[0], np.float64)
    _ref_check(ref().ref_predict_model_file(str(path).encode(), _p(rows), rows.shape[0], rows.shape[1], _p(out)))
    return out


def ref_schedule(jobs, E, T, exec_time, sm, mem, mode=0, budget=0, objective=0, best_effort=0):
    jobs = np.ascontiguousarray(jobs, JOB_DTYPE)
    n = jobs.shape[0]
    out = np.zeros(n, DECISION_DTYPE)
    order = np.zeros(n, np.int64)
    arrs = [np.ascontiguousarray(x, np.float64) for x in (E, T, exec_time)]
    sm = np.ascontiguousarray(sm, np.int32)
    mem = np.ascontiguousarray(mem, np.int32)
    _ref_check(ref().ref_schedule_tables(_p(jobs), n, *[_p(x) for x in arrs], _p(sm), _p(mem), sm.shape[0], mode,
                                         budget, objective, best_effort, _p(out), _p(order)))
    return out, order


def ref_c1_scenario(out_dir, seed=7, stride=2, iters=100, depth=10, n_jobs=100, mode=0, budget=0, objective=0,
                    best_effort=0):
    Path(out_dir).mkdir(parents=True, exist_ok=True)
    _ref_check(ref().ref_c1_scenario(str(out_dir).encode(), seed, stride, iters, depth, n_jobs, mode, budget,
                                     objective, best_effort))
    return load_c1_dir(out_dir)


def load_c1_dir(d):
    d = Path(d)
    meta = np.fromfile(d / "meta.i32", np.int32)
    n_jobs, C_, F, R, K, sm_col, mem_col = (int(x) for x in meta)
    s = dict(n_jobs=n_jobs, n_clocks=C_, n_cols=F, n_records=R, n_cat=K, sm_col=sm_col, mem_col=mem_col)
    s["rows"] = np.fromfile(d / "rows.f64", np.float64).reshape(R, F)
    s["cat_t"] = np.fromfile(d / "cat_t.f64", np.float64).reshape(R, K)
    s["cat_cols"] = np.fromfile(d / "cat_cols.i32", np.int32)
    s["rec_of_clock"] = np.fromfile(d / "rec_of_clock.i32", np.int32).reshape(n_jobs, C_)
    s["sm"] = np.fromfile(d / "sm.i32", np.int32)
    s["mem"] = np.fromfile(d / "mem.i32", np.int32)
    s["arrival"] = np.fromfile(d / "arrival.f64", np.float64)
    s["deadline"] = np.fromfile(d / "deadline.f64", np.float64)
    s["exec"] = np.fromfile(d / "exec.f64", np.float64).reshape(n_jobs, C_)
    s["pred_energy"] = np.fromfile(d / "pred_energy.f64", np.float64).reshape(n_jobs, C_)
    s["pred_time"] = np.fromfile(d / "pred_time.f64", np.float64).reshape(n_jobs, C_)
    s["decisions"] = np.fromfile(d / "decisions.bin", DECISION_DTYPE)
    s["order"] = np.fromfile(d / "order.i64", np.int64)
    s["columns"] = (d / "columns.txt").read_text().split()
    s["model_energy"] = d / "model_energy_gbt.txt"
    s["model_time"] = d / "model_time_gbt.txt"
    return s


def ref_truth_oracle(seed_offset, deadlines):
    deadlines = np.ascontiguousarray(deadlines, np.float64)
    n = deadlines.shape[0]
    E = np.empty((n, 62), np.float64)
    T = np.empty((n, 62), np.float64)
    out = np.zeros(n, DECISION_DTYPE)
    sm = np.empty(62, np.int32)
    _ref_check(ref().ref_truth_oracle(seed_offset, _p(deadlines), _p(E), _p(T), _p(out), _p(sm)))
    return E, T, out, sm


def ref_bench_grid(fe, ft, grid, budgets, n_apps, threads, tables=False):
    """The reference's predict (E, T over materialised candidate rows) +
    schedule_d_dvfs(full_deadline) per app on `threads` host threads; returns
    (seconds, decisions) or, with ``tables``, (seconds, decisions, E, T)."""
    fve, k1 = forest_view(fe)
    fvt, k2 = forest_view(ft)
    rows = np.ascontiguousarray(grid.rows[:n_apps], np.float64)
    cat_t = np.ascontiguousarray(grid.cat_t[:n_apps], np.float64)
    cat_cols = np.ascontiguousarray(grid.cat_cols, np.int32)
    sm = np.ascontiguousarray(grid.sm, np.int32)
    mem = np.ascontiguousarray(grid.mem, np.int32)
    b = np.ascontiguousarray(budgets[:n_apps], np.float64)
    out = np.zeros(n_apps, DECISION_DTYPE)
    E = np.empty((n_apps, sm.shape[0])) if tables else None
    T = np.empty((n_apps, sm.shape[0])) if tables else None
    secs = ref().ref_bench_grid(C.byref(fve), fe.base, fe.learning_rate, C.byref(fvt), ft.base, ft.learning_rate,
                                _p(rows), rows.shape[1], _p(cat_t), _p(cat_cols), cat_cols.shape[0], n_apps, _p(sm),
                                _p(mem), sm.shape[0], grid.sm_col, grid.mem_col, _p(b), threads, _p(out), _p(E),
                                _p(T))
    if secs < 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return (secs, out, E, T) if tables else (secs, out)


def ref_grid_tables(fe, ft, grid, threads=0):
    """E/T candidate tables of every app of `grid` from the reference's own
    predict (record = app; untimed use: deadlines for a CPU sample)."""
    import os

    n = grid.n_apps
    _, dec, E, T = ref_bench_grid(fe, ft, grid, np.ones(n), n, threads or (os.cpu_count() or 1), tables=True)
    return dec, E, T
