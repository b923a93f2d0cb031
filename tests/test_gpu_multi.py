"""GPU: the multi-device C ABI (gd_multi / gd_comm) on the devices
this box has.  With one GPU a group of one runs the same sharding, replica and
gather code as N > 1 minus the NCCL peers; with more GPUs every size up to
the device count is checked.  Decisions and E/T tables must be bit-identical
to single-device gd_grid_select and to the oracle."""
import ctypes as C

import numpy as np
import pytest

import oracle_lib as O
import paper_2004_08177_b200 as gd
from paper_2004_08177_b200 import shard
from paper_2004_08177_b200 import workload as W

pytestmark = pytest.mark.gpu


def _n_devices():
    import torch

    return torch.cuda.device_count()


@pytest.mark.parametrize("n_apps", [1, 97, 3000])
def test_multi_grid_select_matches_single_device_and_oracle(n_apps):
    sc = W.make_scenario("multi", n_apps, "gtx980", 40, 7, seed=n_apps, w_clk=0.1)
    _, _, t0 = O.oracle_grid(sc.energy, sc.time, sc.grid, np.ones(n_apps))
    budgets = W.deadlines_from_times(t0, seed=3)
    want, we, wt = O.oracle_grid(sc.energy, sc.time, sc.grid, budgets)
    for n_dev in sorted({1, _n_devices()}):
        multi = gd.Multi(list(range(n_dev)))
        try:
            src = gd.Model.from_forest(sc.energy, host_only=True)
            src_t = gd.Model.from_forest(sc.time, host_only=True)
            me, mt = multi.replicate(src), multi.replicate(src_t)
            got, e, t = multi.grid_select(me, mt, sc.grid, budgets, return_predictions=True)
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
            assert np.array_equal(e.view(np.int64), we.view(np.int64))
            assert np.array_equal(t.view(np.int64), wt.view(np.int64))
            only = multi.grid_select(me, mt, sc.grid, budgets)  # decisions only
            assert np.array_equal(only.view(np.uint8), want.view(np.uint8))
            for m in me + mt:
                m.close()
        finally:
            multi.close()


def test_multi_general_mode_rec_of_clock():
    sc = W.make_scenario("multi_g", 30, "p100", 20, 6, seed=9, w_clk=0.2)
    rng = np.random.default_rng(1)
    rec = rng.integers(0, 30, size=(30, sc.grid.n_clocks)).astype(np.int32)
    g = W.GridInputs(sc.grid.rows, sc.grid.cat_t, sc.grid.cat_cols, sc.grid.sm, sc.grid.mem, sc.grid.sm_col,
                     sc.grid.mem_col, rec_of_clock=rec)
    budgets = np.full(30, 5.0)
    want, we, wt = O.oracle_grid(sc.energy, sc.time, g, budgets)
    multi = gd.Multi([0])
    try:
        me = multi.replicate(gd.Model.from_forest(sc.energy, host_only=True))
        mt = multi.replicate(gd.Model.from_forest(sc.time, host_only=True))
        got, e, t = multi.grid_select(me, mt, g, budgets, return_predictions=True)
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
        assert np.array_equal(e.view(np.int64), we.view(np.int64))
        assert np.array_equal(t.view(np.int64), wt.view(np.int64))
    finally:
        multi.close()


def test_comm_single_rank_gather_and_model_device_check():
    import torch

    ctx = gd.Context(0)
    comm = gd.Comm(ctx, gd.Comm.make_id(), 1, 0)
    src = torch.arange(24 * 50, dtype=torch.uint8, device="cuda:0") % 251
    dst = torch.zeros_like(src)
    torch.cuda.synchronize()
    comm.gather_decisions(src.data_ptr(), [50], dst.data_ptr(), 0)
    ctx.synchronize()
    assert torch.equal(src, dst)
    with pytest.raises(ValueError):
        comm.gather_decisions(src.data_ptr(), [50, 1], dst.data_ptr(), 0)
    comm.close()
    # a model outlives the context that uploaded it, and serves another
    # context of the same device (no dangling ctx in the model)
    sc = W.make_scenario("life", 20, "gtx980", 10, 5, seed=2)
    other = gd.Context(0)
    me, mt = gd.Model.from_forest(sc.energy, other), gd.Model.from_forest(sc.time, other)
    other.close()
    me.ctx = mt.ctx = ctx
    got = gd.grid_select(me, mt, sc.grid, np.full(20, 9.0))
    want, _, _ = O.oracle_grid(sc.energy, sc.time, sc.grid, np.full(20, 9.0))
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
    ctx.close()


def test_shard_counts_match_library_split():
    # the C side (gd_multi.cpp shard_range) and shard.py split identically
    for n in (0, 1, 97, 10_000_000):
        for g in (1, 2, 3, 8):
            assert sum(shard.shard_counts(n, g)) == n
