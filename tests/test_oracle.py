"""Pin the CPU oracle (oracle/gd_oracle.c) to the reference.

Against the golden fixtures produced by the reference itself
(tests/golden/make_golden.py), and -- where oracle/_ref has been built --
against live calls into the reference's own compiled sources.
"""
import itertools

import numpy as np
import pytest

import oracle_lib as O
from helpers import FIELDS, GOLDEN, bits, c1_combo, c1_small, decisions_equal, golden_forest, parse_model_text
from paper_2004_08177_b200 import workload as W

COMBOS = ["".join(map(str, c)) for c in itertools.product((0, 1), repeat=4)]


@pytest.mark.parametrize("key", ["complete_0", "complete_1", "irregular_0", "irregular_1"])
def test_oracle_predict_matches_reference_golden(key):
    npz = np.load(GOLDEN / "predict.npz")
    f = golden_forest(npz, key, int(key[-1]))
    got = O.oracle_predict(f, npz[f"{key}_rows"])
    assert np.array_equal(bits(got), bits(npz[f"{key}_pred"]))


def test_oracle_energy_clamp_golden():
    # models.cpp:424 -- negative energy predictions clamp to exactly +0.0
    npz = np.load(GOLDEN / "predict.npz")
    f = golden_forest(npz, "neg", 0)
    got = O.oracle_predict(f, npz["neg_rows"])
    assert np.array_equal(bits(got), bits(npz["neg_pred"]))
    assert np.all(bits(got) == 0)


def test_oracle_model_file_golden():
    f = parse_model_text(GOLDEN / "model_time_small.txt")
    npz = np.load(GOLDEN / "model_file_pred.npz")
    assert np.array_equal(bits(O.oracle_predict(f, npz["rows"])), bits(npz["pred"]))


def test_oracle_c1_predictions_golden():
    s = c1_small()
    dec, e, t = O.oracle_grid(s["fe"], s["ft"], s["grid"], s["deadline"])
    assert np.array_equal(bits(e), bits(s["pred_energy"]))
    assert np.array_equal(bits(t), bits(s["pred_time"]))


@pytest.mark.parametrize("tag", COMBOS)
def test_oracle_c1_schedule_golden(tag):
    s = c1_small()
    mode, budget, obj, be = (int(c) for c in tag)
    want, want_order = c1_combo(s, tag)
    got, order = O.oracle_schedule(s["jobs"], s["pred_energy"], s["pred_time"], s["exec"], s["sm"], mode, budget,
                                   obj, be)
    assert decisions_equal(got, want)
    assert np.array_equal(order, want_order)


def test_oracle_c1_default_decisions_golden():
    s = c1_small()
    got, order = O.oracle_schedule(s["jobs"], s["pred_energy"], s["pred_time"], s["exec"], s["sm"])
    assert decisions_equal(got, s["decisions"])
    assert np.array_equal(order, s["order"])


@pytest.mark.parametrize("seed", range(4))
def test_oracle_acceptance1_truth_golden(seed):
    # with the ground truth as predictor, text-mode selection at
    # the full deadline equals oracle_per_job for every job.
    npz = np.load(GOLDEN / "truth.npz")
    got = O.oracle_select(npz[f"s{seed}_E"], npz[f"s{seed}_T"], npz["sm"], npz[f"s{seed}_deadline"])
    assert decisions_equal(got, npz[f"s{seed}_decisions"])


def test_spec_examples():
    # clocks {low: (100 W.s, 10 s), high: (150 W.s, 5 s)}
    E = np.array([[100.0, 150.0]])
    T = np.array([[10.0, 5.0]])
    sm = np.array([500, 1000], np.int32)
    for dl, want in ((8.0, 1), (12.0, 0), (3.0, -1)):
        d = O.oracle_select(E, T, sm, [dl])
        assert d["clock_index"][0] == want
        assert d["status"][0] == (0 if want >= 0 else 1)


# ---- live reference (oracle/_ref) --------------------------------------------

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("leaf_prob,w_clk", [(0.0, 0.04), (0.3, 0.25)])
def test_oracle_predict_live_reference(leaf_prob, w_clk):
    sc = W.make_scenario("t", 16, "gtx980", 40, 6, seed=3, w_clk=w_clk, leaf_prob=leaf_prob)
    rows = np.repeat(sc.grid.rows, 5, axis=0)
    rows[:, W.SM_COL] = np.resize(sc.grid.sm, rows.shape[0])
    rows[:, W.MEM_COL] = np.resize(sc.grid.mem, rows.shape[0])
    for f in (sc.energy, sc.time):
        assert np.array_equal(bits(O.oracle_predict(f, rows)), bits(O.ref_predict(f, rows)))


@needs_ref
def test_oracle_c1_full_scale_live(tmp_path):
    # The BASELINE configs[0] shape: 100 trees depth 10, 62 clocks, 100 jobs.
    s = O.ref_c1_scenario(tmp_path, seed=7, iters=100, depth=10, n_jobs=100)
    fe, ft = parse_model_text(s["model_energy"]), parse_model_text(s["model_time"])
    g = W.GridInputs(s["rows"], s["cat_t"], s["cat_cols"], s["sm"], s["mem"], s["sm_col"], s["mem_col"],
                     s["rec_of_clock"])
    _, e, t = O.oracle_grid(fe, ft, g, s["deadline"])
    assert np.array_equal(bits(e), bits(s["pred_energy"]))
    assert np.array_equal(bits(t), bits(s["pred_time"]))
    jobs = np.zeros(s["n_jobs"], O.JOB_DTYPE)
    jobs["arrival_s"], jobs["deadline_s"] = s["arrival"], s["deadline"]
    jobs["app_rank"] = jobs["app_index"] = np.arange(s["n_jobs"])
    got, order = O.oracle_schedule(jobs, e, t, s["exec"], s["sm"])
    assert decisions_equal(got, s["decisions"])
    assert np.array_equal(order, s["order"])


@needs_ref
def test_oracle_edf_ties_live():
    # Equal absolute deadlines / arrivals force the (abs, arrival, app_id) tie rules.
    rng = np.random.default_rng(4)
    n, A, Cn = 60, 12, 8
    jobs = np.zeros(n, O.JOB_DTYPE)
    jobs["arrival_s"] = rng.integers(0, 5, size=n).astype(np.float64)
    jobs["deadline_s"] = rng.integers(1, 4, size=n).astype(np.float64)
    jobs["app_rank"] = rng.permutation(n)
    jobs["app_index"] = rng.integers(0, A, size=n)
    E = rng.integers(1, 4, size=(A, Cn)).astype(np.float64)
    T = rng.integers(1, 4, size=(A, Cn)).astype(np.float64) * 0.25
    X = T.copy()
    sm, mem = np.arange(100, 100 + Cn, dtype=np.int32), np.full(Cn, 700, np.int32)
    for mode, budget, obj, be in itertools.product((0, 1), repeat=4):
        want, wo = O.ref_schedule(jobs, E, T, X, sm, mem, mode, budget, obj, be)
        got, go = O.oracle_schedule(jobs, E, T, X, sm, mode, budget, obj, be)
        assert decisions_equal(got, want) and np.array_equal(go, wo)


@needs_ref
@pytest.mark.parametrize("seed", range(12))
def test_oracle_fuzz_live_reference(seed):
    """Random ensembles (depth, irregularity, clock-split rate), rows with NaN
    and extreme feature values, and random E/T tables with heavy ties through
    every selection option: the oracle and the reference's own compiled code
    agree bit for bit."""
    rng = np.random.default_rng(500 + seed)
    sc = W.make_scenario("fz", 12, "gtx980", int(rng.integers(1, 40)), int(rng.integers(1, 11)), seed=seed,
                         w_clk=float(rng.choice([0.0, 0.1, 0.4])), leaf_prob=float(rng.choice([0.0, 0.3])))
    rows = np.repeat(sc.grid.rows, 4, axis=0)
    rows[:, W.SM_COL] = np.resize(sc.grid.sm, rows.shape[0])
    rows[:, W.MEM_COL] = np.resize(sc.grid.mem, rows.shape[0])
    mask = rng.random(rows.shape) < 0.05
    rows[mask] = np.nan
    rows[rng.random(rows.shape) < 0.02] = 1e300
    rows[rng.random(rows.shape) < 0.02] = -1e300
    for f in (sc.energy, sc.time):
        assert np.array_equal(bits(O.oracle_predict(f, rows)), bits(O.ref_predict(f, rows)))
    # selection + EDF over tie-heavy tables
    n, A, Cn = 40, 9, int(rng.integers(1, 20))
    jobs = np.zeros(n, O.JOB_DTYPE)
    jobs["arrival_s"] = rng.integers(0, 6, size=n).astype(np.float64)
    jobs["deadline_s"] = rng.integers(1, 5, size=n).astype(np.float64)
    jobs["app_rank"] = rng.permutation(n)
    jobs["app_index"] = rng.integers(0, A, size=n)
    E = rng.integers(1, 4, size=(A, Cn)).astype(np.float64)
    T = rng.integers(1, 5, size=(A, Cn)).astype(np.float64) * 0.5
    X = T * rng.choice([0.5, 1.0, 1.5], size=(A, Cn))
    # a valid catalog: unique (sm, mem) pairs in clock_catalog order (mem, sm ascending)
    pairs = sorted({(int(m), int(x)) for m, x in zip(rng.choice([405, 810, 3505], size=Cn),
                                                     rng.integers(300, 1500, size=Cn))})
    Cn = len(pairs)
    E, T, X = E[:, :Cn], T[:, :Cn], X[:, :Cn]
    sm = np.array([x for _, x in pairs], np.int32)
    mem = np.array([m for m, _ in pairs], np.int32)
    for mode, budget, obj, be in itertools.product((0, 1), repeat=4):
        want, worder = O.ref_schedule(jobs, E, T, X, sm, mem, mode, budget, obj, be)
        got, gorder = O.oracle_schedule(jobs, E, T, X, sm, mode, budget, obj, be)
        assert decisions_equal(got, want), (seed, mode, budget, obj, be)
        assert np.array_equal(gorder, worder)
