"""N > 1 host logic on CPU: row sharding + the single decision gather
(paper_2004_08177_b200/shard.py) with world_size 2 over gloo.

Each rank computes the decisions of its contiguous app shard (with the oracle
standing in for the device kernel, which this CPU test cannot run), the ranks
all-gather the 24-byte records, and every rank must hold exactly the
decisions of the whole batch in app order.
"""
import os
import socket

import numpy as np
import pytest

from paper_2004_08177_b200 import shard
from paper_2004_08177_b200 import workload as W


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_apps, result_dir):
    import torch
    import torch.distributed as dist

    import oracle_lib as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = W.make_scenario("mg", n_apps, "p100", 12, 5, seed=21)
    budgets = np.full(n_apps, 7.0)
    lo, hi = shard.shard_range(n_apps, rank, world)
    dec, _, _ = O.oracle_grid(sc.energy, sc.time, sc.grid, budgets, app_slice=(lo, hi))
    local = torch.from_numpy(dec.view(np.uint8).copy())
    full = shard.gather_decisions(local, n_apps, world)
    np.save(os.path.join(result_dir, f"rank{rank}.npy"), full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_cover_batch():
    for n in (0, 1, 7, 64, 10_001):
        for world in (1, 2, 3, 8):
            ranges = [shard.shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.shard_range(10, 2, 2)


@pytest.mark.parametrize("n_apps", [37, 64])
def test_gather_decisions_world2_gloo(tmp_path, n_apps):
    import torch.multiprocessing as mp

    import oracle_lib as O

    port = _free_port()
    mp.start_processes(_worker, args=(2, port, n_apps, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    sc = W.make_scenario("mg", n_apps, "p100", 12, 5, seed=21)
    want, _, _ = O.oracle_grid(sc.energy, sc.time, sc.grid, np.full(n_apps, 7.0))
    for r in range(2):
        got = np.load(tmp_path / f"rank{r}.npy").view(O.DECISION_DTYPE)
        assert got.shape == (n_apps,)
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


def _bench_worker(rank, world, port, n_apps, result_dir):
    """bench.py's own sharded path, CPU-side: each rank builds ITS shard of the
    configs[1]-shape workload with bench.make_inputs (chunk-seeded rows), the
    oracle stands in for the kernels, and the decisions reach rank 0 through
    the gather-to-root mirror of gd_gather_decisions."""
    import sys
    from pathlib import Path

    import torch
    import torch.distributed as dist

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    import oracle_lib as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, per_rank, total = bench.workload_config("c4", world, apps=n_apps)
    cfg = dict(cfg, n_trees=24, depth=6)  # small ensembles: the oracle stands in for the device
    lo, hi = shard.shard_range(total, rank, world)
    sc = bench.make_inputs(cfg, total, (lo, hi))
    dec, _, _ = O.oracle_grid(sc.energy, sc.time, sc.grid, np.full(hi - lo, 3.0))
    full = shard.gather_decisions_to_root(torch.from_numpy(dec.view(np.uint8).copy()), total, world)
    if rank == 0:
        np.save(os.path.join(result_dir, "root.npy"), full.numpy())
    else:
        assert full is None
    dist.barrier()
    dist.destroy_process_group()


def test_bench_sharded_path_world2_gloo(tmp_path):
    import sys
    from pathlib import Path

    import torch.multiprocessing as mp

    import oracle_lib as O

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench

    n_apps = 45
    port = _free_port()
    mp.start_processes(_bench_worker, args=(2, port, n_apps, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    cfg, _, total = bench.workload_config("c4", 1, apps=n_apps)
    cfg = dict(cfg, n_trees=24, depth=6)
    sc = bench.make_inputs(cfg, total, (0, total))  # the one-rank batch
    want, _, _ = O.oracle_grid(sc.energy, sc.time, sc.grid, np.full(total, 3.0))
    got = np.load(tmp_path / "root.npy").view(O.DECISION_DTYPE)
    assert got.shape == (total,)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
    assert shard.shard_counts(total, 2) == [22, 23]
