"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

    python tests/golden/make_golden.py

Runs the reference's own code (compiled from /root/reference/proj/src by
oracle/Makefile into oracle/_ref/libgpudvfs_ref.so, driven through
oracle/ref_shim.cpp) and stores its outputs:

* c1_small/        the paper-scale production path at reduced size
                   (cli.cpp:400-481 equivalent: fit_gbt -> save/load model
                   files -> select_k clusters -> make_model_predictor ->
                   schedule_d_dvfs), with every GPU-path input dumped and the
                   reference's per-(job, clock) predictions and decisions, plus
                   the reference's decisions for every SchedulerOptions combo.
* predict.npz      synthetic forests + rows and models::predict's outputs
                   (models.cpp:395-428); a model file written by save_model.
* truth.npz        acceptance #1 material: the synthetic ground
                   truth E/T over the P100 catalog and oracle_per_job's
                   decisions (scheduler.cpp:257-281).
"""
from __future__ import annotations

import itertools
import shutil
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))

import oracle_lib as O  # noqa: E402
from paper_2004_08177_b200 import workload as W  # noqa: E402

OPTION_COMBOS = list(itertools.product((0, 1), (0, 1), (0, 1), (0, 1)))  # mode, budget, objective, best_effort


def make_c1_small():
    d = HERE / "c1_small"
    if d.exists():
        shutil.rmtree(d)
    s = O.ref_c1_scenario(d, seed=11, stride=2, iters=24, depth=6, n_jobs=40)
    jobs = np.zeros(s["n_jobs"], O.JOB_DTYPE)
    jobs["arrival_s"], jobs["deadline_s"] = s["arrival"], s["deadline"]
    jobs["app_rank"] = np.arange(s["n_jobs"])
    jobs["app_index"] = np.arange(s["n_jobs"])
    for mode, budget, obj, be in OPTION_COMBOS:
        dec, order = O.ref_schedule(jobs, s["pred_energy"], s["pred_time"], s["exec"], s["sm"], s["mem"], mode,
                                    budget, obj, be)
        tag = f"{mode}{budget}{obj}{be}"
        dec.tofile(d / f"decisions_{tag}.bin")
        order.tofile(d / f"order_{tag}.i64")
    print("c1_small:", s["n_jobs"], "jobs,", (s["decisions"]["status"] == 0).sum(), "scheduled")


def make_predict():
    rng = np.random.default_rng(5)
    sm, mem = W.catalog_p100()
    cols = W._ColumnModel(rng, W.N_COLS, W.CAT_COLS, sm, mem, W.SM_COL, W.MEM_COL)
    out = {}
    for name, kw in {"complete": dict(n_trees=16, depth=4, leaf_prob=0.0),
                     "irregular": dict(n_trees=16, depth=7, leaf_prob=0.3)}.items():
        for target in (0, 1):
            f = W.make_forest(cols, seed=100 + target, target=target, w_clk=0.1, **kw)
            rows, _ = W.make_rows(cols, 64, 200 + target, 1189, 715)
            rows[:, W.SM_COL] = sm[rng.integers(0, len(sm), size=64)]
            p = O.ref_predict(f, rows)
            key = f"{name}_{target}"
            for fld in ("tree_offsets", "feature", "threshold", "left", "right", "leaf_value"):
                out[f"{key}_{fld}"] = getattr(f, fld)
            out[f"{key}_base"] = np.array([f.base])
            out[f"{key}_lr"] = np.array([f.learning_rate])
            out[f"{key}_rows"] = rows
            out[f"{key}_pred"] = p
    # Energy clamp: a forest whose prediction goes negative must give exactly 0.0.
    f = W.make_forest(cols, n_trees=4, depth=3, target=0, seed=9)
    f.base = -1.0e4
    rows, _ = W.make_rows(cols, 8, 9, 1189, 715)
    out["neg_pred"] = O.ref_predict(f, rows)
    for fld in ("tree_offsets", "feature", "threshold", "left", "right", "leaf_value"):
        out[f"neg_{fld}"] = getattr(f, fld)
    out["neg_rows"] = rows
    out["neg_base"] = np.array([f.base])
    out["neg_lr"] = np.array([f.learning_rate])
    np.savez_compressed(HERE / "predict.npz", **out)
    # A model file written by the reference's save_model (preorder, %.17g).
    f = W.make_forest(cols, n_trees=6, depth=5, target=1, seed=77, leaf_prob=0.25)
    O.ref_save_forest(f, HERE / "model_time_small.txt")
    rows, _ = W.make_rows(cols, 32, 78, 1189, 715)
    np.savez_compressed(HERE / "model_file_pred.npz", rows=rows,
                        pred=O.ref_predict_model_file(HERE / "model_time_small.txt", rows))
    print("predict.npz written")


def make_truth():
    out = {}
    for seed in range(4):
        rng = np.random.default_rng(1000 + seed)
        # deadlines: factor in (1, 2) x the default-clock truth time, ~10% infeasible
        E, T, _, sm = O.ref_truth_oracle(seed, np.ones(12))
        default_idx = int(np.nonzero(sm == 1189)[0][0])
        dl = rng.uniform(1.0, 2.0, size=12) * T[:, default_idx]
        bad = rng.random(12) < 0.1
        dl[bad] = T[bad].min(axis=1) * 0.5
        E, T, dec, sm = O.ref_truth_oracle(seed, dl)
        out[f"s{seed}_E"], out[f"s{seed}_T"], out[f"s{seed}_deadline"] = E, T, dl
        out[f"s{seed}_decisions"] = dec
        out["sm"] = sm
    np.savez_compressed(HERE / "truth.npz", **out)
    print("truth.npz written")


if __name__ == "__main__":
    O.build_oracle(ref=True)
    if not O.ref_available():
        sys.exit("oracle/_ref not built (needs /root/reference)")
    make_c1_small()
    make_predict()
    make_truth()
