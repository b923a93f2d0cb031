"""CPU-side checks of the native library: exports, parser, packer, EDF host loop.

None of these launch kernels; they run without a GPU.
"""
import itertools
import re
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
import paper_2004_08177_b200 as gd
from helpers import GOLDEN, c1_combo, c1_small, decisions_equal, parse_model_text
from paper_2004_08177_b200 import _capi
from paper_2004_08177_b200 import workload as W

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "gdvfs.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(gd_[a-z_0-9]+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _capi.lib()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_capi.SIGNATURES), set(names) ^ set(_capi.SIGNATURES)
    assert b"sm_100a" in lib.gd_version()


def test_no_device_fails_loudly():
    try:
        ctx = gd.Context(0)
    except gd.GdError as e:
        assert e.code == _capi.GD_ERR_CUDA
        return
    ctx.close()
    pytest.skip("a GPU is present")


def test_model_file_parse_matches_reference_layout():
    path = GOLDEN / "model_time_small.txt"
    m = gd.Model.load_file(path, host_only=True)
    want = parse_model_text(path)
    got = m.export()
    for f in ("tree_offsets", "feature", "threshold", "left", "right", "leaf_value"):
        assert np.array_equal(getattr(got, f), getattr(want, f)), f
    assert m.target == 1 and m.kind == 2 and m.n_trees == want.n_trees
    assert m.base == want.base and m.learning_rate == want.learning_rate
    assert len(m.columns) == want.n_cols


def test_c1_model_files_parse():
    s = c1_small()
    for path, f in ((s["model_energy"], s["fe"]), (s["model_time"], s["ft"])):
        m = gd.Model.load_file(path, host_only=True)
        assert m.columns == s["columns"]
        got = m.export()
        assert np.array_equal(got.threshold.view(np.int64), f.threshold.view(np.int64))
        assert np.array_equal(got.leaf_value.view(np.int64), f.leaf_value.view(np.int64))
        assert m.max_depth <= 6


def test_model_file_errors(tmp_path):
    # models.cpp:639-714 error kinds and messages
    missing = tmp_path / "nope.txt"
    with pytest.raises(gd.MissingArtifactError, match=re.escape(f"cannot open model '{missing}'")):
        gd.Model.load_file(missing, host_only=True)
    bad = tmp_path / "bad.txt"
    bad.write_text("gpudvfs-model 2\n")
    with pytest.raises(gd.DataError, match="not a gpudvfs-model v1 file"):
        gd.Model.load_file(bad, host_only=True)
    good = (GOLDEN / "model_time_small.txt").read_text()
    trunc = tmp_path / "trunc.txt"
    trunc.write_text(good[: len(good) // 2].rsplit("\n", 1)[0] + "\nnode 3")
    with pytest.raises(gd.DataError, match="truncated model file|expected 'node'"):
        gd.Model.load_file(trunc, host_only=True)
    kind = tmp_path / "kind.txt"
    kind.write_text(good.replace("kind gbt", "kind forest"))
    with pytest.raises(ValueError, match="unknown model kind 'forest'"):
        gd.Model.load_file(kind, host_only=True)
    target = tmp_path / "target.txt"
    target.write_text(good.replace("target time", "target power"))
    with pytest.raises(ValueError, match="unknown target 'power'"):
        gd.Model.load_file(target, host_only=True)
    # comment stamps are skipped (textio.hpp:39-44)
    stamped = tmp_path / "stamped.txt"
    stamped.write_text("# gpudvfs config_hash=1 seed=2\n" + good)
    assert gd.Model.load_file(stamped, host_only=True).n_trees == parse_model_text(GOLDEN / "model_time_small.txt").n_trees


def small_forest():
    sc = W.make_scenario("p", 4, "p100", 3, 3, seed=1)
    return sc.energy


@pytest.mark.parametrize("corrupt", ["child_range", "shared_child", "cycle", "feature"])
def test_packer_rejects_malformed_trees(corrupt):
    f = small_forest()
    f.left = f.left.copy()
    f.feature = f.feature.copy()
    if corrupt == "child_range":
        f.left[0] = 10_000
    elif corrupt == "shared_child":
        f.left[0] = f.right[0]
    elif corrupt == "cycle":
        f.left[1] = 0
    else:
        f.feature[0] = W.N_COLS
    with pytest.raises(gd.DataError):
        gd.Model.from_forest(f, host_only=True)


def test_packer_accepts_level_and_preorder():
    f = small_forest()
    m = gd.Model.from_forest(f, host_only=True)
    assert m.max_depth == 3 and m.n_trees == 3


# ---- EDF host loop (gd_schedule_edf) -----------------------------------------

@pytest.mark.parametrize("tag", ["".join(map(str, c)) for c in itertools.product((0, 1), repeat=4)])
def test_edf_matches_reference_c1_golden(tag):
    s = c1_small()
    mode, budget, obj, be = (int(c) for c in tag)
    want, want_order = c1_combo(s, tag)
    opts = gd.SchedulerOptions(mode=["text", "literal"][mode], budget=["remaining", "full"][budget],
                               objective=["energy", "power"][obj], best_effort_fallback=bool(be))
    got, order = gd.schedule_d_dvfs(s["jobs"], s["pred_energy"], s["pred_time"], s["sm"], s["exec"], opts)
    assert decisions_equal(got, want)
    assert np.array_equal(order, want_order)


@pytest.mark.parametrize("seed", range(6))
def test_edf_ties_match_oracle(seed):
    rng = np.random.default_rng(seed)
    n, A, Cn = 200, 15, 9
    jobs = np.zeros(n, O.JOB_DTYPE)
    jobs["arrival_s"] = rng.integers(0, 8, size=n).astype(np.float64)
    jobs["deadline_s"] = rng.integers(1, 5, size=n).astype(np.float64) * 0.5
    jobs["app_rank"] = rng.permutation(n)
    jobs["app_index"] = rng.integers(-1, A, size=n)  # -1: missing correlated data
    E = rng.integers(0, 3, size=(A, Cn)).astype(np.float64)
    T = rng.integers(1, 4, size=(A, Cn)).astype(np.float64) * 0.25
    X = T * rng.uniform(0.5, 1.5, size=T.shape)
    sm = np.sort(rng.choice(np.arange(300, 2000), Cn, replace=False)).astype(np.int32)
    for mode, budget, obj, be in itertools.product((0, 1), repeat=4):
        want, wo = O.oracle_schedule(jobs, E, T, X, sm, mode, budget, obj, be)
        opts = gd.SchedulerOptions(mode=["text", "literal"][mode], budget=["remaining", "full"][budget],
                                   objective=["energy", "power"][obj], best_effort_fallback=bool(be))
        got, go = gd.schedule_d_dvfs(jobs, E, T, sm, X, opts)
        assert decisions_equal(got, want), (mode, budget, obj, be)
        assert np.array_equal(go, wo)


@pytest.mark.parametrize("seed", range(4))
def test_edf_frontier_queries_match_scan(seed):
    # gd_schedule_edf_frontier (binary search on the per-app frontier) makes
    # the same decisions as the O(C) scan for every option combination; the
    # frontier here is the plain restatement (the GPU test checks the kernel).
    from helpers import frontier_ref
    rng = np.random.default_rng(100 + seed)
    n, A, Cn = 300, 20, 33
    jobs = np.zeros(n, O.JOB_DTYPE)
    jobs["arrival_s"] = rng.integers(0, 8, size=n).astype(np.float64)
    jobs["deadline_s"] = rng.integers(1, 9, size=n).astype(np.float64) * 0.5
    jobs["app_rank"] = rng.permutation(n)
    jobs["app_index"] = rng.integers(-1, A, size=n)
    E = rng.integers(0, 4, size=(A, Cn)).astype(np.float64) + 1.0
    T = rng.integers(1, 6, size=(A, Cn)).astype(np.float64) * 0.25
    E[3, 4] = np.nan  # a non-finite row falls back to the scan
    X = T * rng.uniform(0.5, 1.5, size=T.shape)
    sm = np.sort(rng.integers(300, 2000, size=Cn)).astype(np.int32)  # duplicate sm values allowed
    for mode, budget, obj, be in itertools.product((0, 1), repeat=4):
        opts = gd.SchedulerOptions(mode=["text", "literal"][mode], budget=["remaining", "full"][budget],
                                   objective=["energy", "power"][obj], best_effort_fallback=bool(be))
        want, wo = gd.schedule_d_dvfs(jobs, E, T, sm, X, opts)
        got, go = gd.schedule_d_dvfs(jobs, E, T, sm, X, opts, front=frontier_ref(E, T, sm, obj))
        assert decisions_equal(got, want) and np.array_equal(go, wo), (mode, budget, obj, be)


def test_edf_empty_workload():
    out, order = gd.schedule_d_dvfs(np.zeros(0, O.JOB_DTYPE), np.zeros((0, 3)), np.zeros((0, 3)),
                                    np.array([1, 2, 3], np.int32), np.zeros((0, 3)))
    assert out.shape == (0,) and order.shape == (0,)
