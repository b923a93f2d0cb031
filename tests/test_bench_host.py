"""bench.py host logic on CPU: config scaling modes and the chunked on-device
deadline rule (run here on CPU tensors) against workload.deadlines_from_times."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2004_08177_b200 import workload as W  # noqa: E402


def test_workload_config_scaling():
    cfg, per_rank, total = bench.workload_config("c2", 4)
    assert per_rank == W.CONFIGS["c2"]["n_apps"] and total == 4 * per_rank
    cfg, per_rank, total = bench.workload_config("c4", 8)
    assert total == W.CONFIGS["c4"]["n_apps"] and per_rank == -(-total // 8)
    cfg, per_rank, total = bench.workload_config("c4", 1, apps=1000)
    assert (per_rank, total) == (1000, 1000)


def test_chunked_deadlines_match_reference_rule():
    rng = np.random.default_rng(0)
    times = rng.uniform(1.0, 9.0, size=(1000, 267))
    times[:, 5] = times[:, 7]  # ties
    want = W.deadlines_from_times(times, seed=77)
    r = np.random.default_rng(77)
    q = r.uniform(0.1, 0.9, size=1000)
    bad = r.random(size=1000) < 0.05
    idx = np.minimum((q * 266).astype(np.int64), 266)
    got = np.concatenate([bench.deadline_rows(torch.from_numpy(times[lo:lo + 300]), idx[lo:lo + 300],
                                              bad[lo:lo + 300]) for lo in range(0, 1000, 300)])
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
