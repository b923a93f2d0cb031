"""Host-side logic of the Python mirror that needs no GPU: the cached C
gd_grid struct (configs[4] latency path) must follow every change of the
GridInputs it was built from, and the fast data pointers must equal numpy's."""
import ctypes as C

import numpy as np

import paper_2004_08177_b200 as gd
from paper_2004_08177_b200 import workload as W


def _grid(n=16, seed=0):
    rng = np.random.default_rng(seed)
    return W.GridInputs(rng.random((n, 50)), rng.random((n, 2)), np.array([0, 3], np.int32),
                        np.arange(100, 367, dtype=np.int32), np.full(267, 877, np.int32), 42, 25)


def _struct(grid, budgets):
    keep = []
    return gd._grid_struct(grid, budgets, keep), keep


def test_fast_pointer_matches_numpy():
    for a in (np.zeros((3, 5)), np.arange(7, dtype=np.int32), np.zeros(0)):
        assert gd._ptr(a) == a.ctypes.data
    ro = np.ones(4)
    ro.setflags(write=False)
    assert gd._ptr(ro) == ro.ctypes.data
    assert gd._ptr(None) is None


def test_grid_struct_cache_follows_inputs():
    g = _grid()
    b1, b2 = np.ones(16), np.full(16, 2.0)
    s1, _ = _struct(g, b1)
    s2, _ = _struct(g, b2)  # cached: only the budgets pointer differs
    assert s2.rows == s1.rows and s2.budgets == gd._ptr(b2) != s1.budgets
    assert "_gd_struct" in g.__dict__
    # in-place edits keep the same memory: the cached pointers stay valid
    g.rows[0, 0] = 123.0
    s3, _ = _struct(g, b1)
    assert s3.rows == gd._ptr(g.rows)
    # a reassigned field (new array, new shape) rebuilds the struct
    g.rows = np.ascontiguousarray(np.vstack([g.rows, g.rows]))
    g.cat_t = np.ascontiguousarray(np.vstack([g.cat_t, g.cat_t]))
    s4, _ = _struct(g, np.ones(32))
    assert s4.rows == gd._ptr(g.rows) and s4.n_apps == 32 and s4.n_records == 32
    g.sm_col = 7
    s5, _ = _struct(g, np.ones(32))
    assert s5.sm_col == 7


def test_grid_struct_not_cached_for_converted_copies():
    g = _grid()
    g.sm = g.sm.astype(np.int64)  # converted to int32 per call: a copy, never cached
    s, keep = _struct(g, np.ones(16))
    assert "_gd_struct" not in g.__dict__
    assert s.sm_clock != g.sm.ctypes.data
    sm_copy = next(a for a in keep if a is not None and a.dtype == np.int32 and a.shape == (267,) and a is not g.mem)
    assert C.c_int32.from_address(s.sm_clock).value == int(g.sm[0]) == int(sm_copy[0])
