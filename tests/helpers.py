"""Shared test helpers: golden-fixture loaders and small synthetic cases."""
from __future__ import annotations

from pathlib import Path

import numpy as np

import oracle_lib as O
from paper_2004_08177_b200 import workload as W

GOLDEN = Path(__file__).resolve().parent / "golden"
FIELDS = ("tree_offsets", "feature", "threshold", "left", "right", "leaf_value")


def golden_forest(npz, key, target, n_cols=W.N_COLS):
    return W.Forest(*(npz[f"{key}_{f}"] for f in FIELDS), float(npz[f"{key}_base"][0]) if f"{key}_base" in npz
                    else 0.0, float(npz[f"{key}_lr"][0]) if f"{key}_lr" in npz else 0.1, target, n_cols)


def parse_model_text(path) -> W.Forest:
    """Independent Python reading of a "gpudvfs-model 1" file (models.cpp:639-708)."""
    toks = Path(path).read_text().split()
    i = 2
    target = toks[i + 3]
    i += 6
    ncol = int(toks[i + 1])
    i += 2 + 2 * ncol
    base, lr, ntree = float(toks[i + 1]), float(toks[i + 3]), int(toks[i + 5])
    i += 6
    off, f, th, l, r, lv = [0], [], [], [], [], []
    for _ in range(ntree):
        n = int(toks[i + 1])
        i += 2
        for _ in range(n):
            f.append(int(toks[i + 1]))
            th.append(float(toks[i + 2]))
            l.append(int(toks[i + 3]))
            r.append(int(toks[i + 4]))
            lv.append(float(toks[i + 5]))
            i += 6
        off.append(len(f))
    return W.Forest(np.array(off, np.int64), np.array(f, np.int32), np.array(th), np.array(l, np.int32),
                    np.array(r, np.int32), np.array(lv), base, lr, 0 if target == "energy" else 1, ncol)


def c1_small():
    s = O.load_c1_dir(GOLDEN / "c1_small")
    s["fe"] = parse_model_text(s["model_energy"])
    s["ft"] = parse_model_text(s["model_time"])
    s["grid"] = W.GridInputs(s["rows"], s["cat_t"], s["cat_cols"], s["sm"], s["mem"], s["sm_col"], s["mem_col"],
                             s["rec_of_clock"])
    jobs = np.zeros(s["n_jobs"], O.JOB_DTYPE)
    jobs["arrival_s"], jobs["deadline_s"] = s["arrival"], s["deadline"]
    jobs["app_rank"] = np.arange(s["n_jobs"])
    jobs["app_index"] = np.arange(s["n_jobs"])
    s["jobs"] = jobs
    return s


def c1_combo(s, tag):
    d = GOLDEN / "c1_small"
    return np.fromfile(d / f"decisions_{tag}.bin", O.DECISION_DTYPE), np.fromfile(d / f"order_{tag}.i64", np.int64)


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def decisions_equal(a, b):
    return (np.array_equal(a["clock_index"], b["clock_index"]) and np.array_equal(a["status"], b["status"])
            and np.array_equal(a["note"], b["note"]) and np.array_equal(bits(a["energy_ws"]), bits(b["energy_ws"]))
            and np.array_equal(bits(a["time_s"]), bits(b["time_s"])))


def tie_tables(rng, n_apps, n_clocks, levels=4):
    """E/T tables with heavy exact ties (few distinct values) to pin tie-breaks."""
    E = rng.integers(0, levels, size=(n_apps, n_clocks)).astype(np.float64) * 10.0 + 5.0
    T = rng.integers(0, levels, size=(n_apps, n_clocks)).astype(np.float64) * 0.5 + 1.0
    return E, T


def frontier_ref(E, T, sm, objective=0):
    """Plain restatement of gd_frontier (test reference): per app the
    candidates sorted by (T, E, index), the prefix argmin of select_text's
    key (objective, T, sm, index), the best-effort index (-2 if non-finite)."""
    A, Cn = E.shape
    ts = np.empty((A, Cn))
    best = np.empty((A, Cn), np.int32)
    first = np.empty(A, np.int32)
    for a in range(A):
        order = sorted(range(Cn), key=lambda c: (T[a, c], E[a, c], c))
        ts[a] = T[a, order]
        cur = None
        for k, c in enumerate(order):
            obj = E[a, c] / max(T[a, c], 1e-12) if objective else E[a, c]
            key = (obj, T[a, c], sm[c], c)
            if cur is None or key < cur[0]:
                cur = (key, c)
            best[a, k] = cur[1]
        first[a] = order[0] if np.all(np.isfinite(E[a])) and np.all(np.isfinite(T[a])) else -2
    return ts, best, first
