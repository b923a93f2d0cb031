"""GPU training: gd_fit_gbt against the reference's own
models::fit_gbt (oracle/_ref), node for node -- tree shapes, node order,
features, thresholds and leaf values bit-identical -- on the paper-scale C1
catalog (100 trees x depth 10, the facade's production configuration) and on
synthetic matrices with ties, constant columns and pure nodes."""
import numpy as np
import pytest

import oracle_lib as O
import paper_2004_08177_b200 as gd

pytestmark = pytest.mark.gpu


def _same_forest(got, want):
    for f in ("tree_offsets", "feature", "left", "right"):
        assert np.array_equal(getattr(got, f), getattr(want, f)), f
    for f in ("threshold", "leaf_value"):
        assert np.array_equal(getattr(got, f).view(np.int64), getattr(want, f).view(np.int64)), f
    assert np.float64(got.base).view(np.int64) == np.float64(want.base).view(np.int64)


@pytest.fixture(scope="module")
def ctx():
    c = gd.Context(0)
    yield c
    c.close()


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("target", [0, 1])
def test_fit_gbt_c1_catalog_node_for_node(ctx, target):
    rows, targets = O.ref_c1_train(seed=7, stride=2, target=target)
    want = O.ref_fit_gbt(rows, targets, 100, 10, 0.1, 3.0, 7, target)
    m = gd.fit_gbt(rows, targets, 100, 10, 0.1, 3.0, 7, target, ctx=ctx)
    _same_forest(m.export(), want)
    # and the trained model predicts through K1 exactly like the reference
    assert np.array_equal(m.predict(rows).view(np.int64), O.ref_predict(want, rows).view(np.int64))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(6))
def test_fit_gbt_synthetic_vs_reference(ctx, seed):
    rng = np.random.default_rng(seed)
    n, p = int(rng.integers(1, 700)), int(rng.integers(1, 9))
    rows = rng.normal(size=(n, p))
    rows[:, 0] = np.round(rows[:, 0], 1)        # heavy ties
    if p > 2:
        rows[:, 2] = 3.25                       # a constant column
    targets = rows @ rng.normal(size=p) + rng.normal(scale=0.1, size=n)
    if seed % 3 == 0:
        targets[: n // 2] = 1.5                 # pure regions
    iters, depth = int(rng.integers(0, 25)), int(rng.integers(1, 9))
    lr, l2 = float(rng.uniform(0.05, 1.0)), float(rng.choice([0.0, 1.0, 3.0]))
    want = O.ref_fit_gbt(rows, targets, iters, depth, lr, l2, seed, 0)
    got = gd.fit_gbt(rows, targets, iters, depth, lr, l2, seed, 0, ctx=ctx).export()
    _same_forest(got, want)


def test_fit_gbt_config_errors(ctx):
    rows, t = np.ones((4, 2)), np.arange(4.0)
    for kw, msg in [(dict(depth=0), "depth must be >= 1"), (dict(learning_rate=0.0), "learning_rate"),
                    (dict(iterations=-1), "iterations must be >= 0"), (dict(l2_leaf_reg=-1.0), "l2_leaf_reg")]:
        with pytest.raises(ValueError, match=msg):
            gd.fit_gbt(rows, t, ctx=ctx, **kw)
    with pytest.raises(ValueError, match="empty training matrix"):
        gd.fit_gbt(np.ones((0, 2)), np.ones(0), ctx=ctx)
