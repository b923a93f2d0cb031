"""K1 (models::predict drop-in) throughput on B200: rows/s for the configs[1]
ensembles (500 trees, depth 8) over materialised rows, vs the reference's
predict on one host core (oracle/_ref) for a small sample."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2004_08177_b200 as gd  # noqa: E402
from paper_2004_08177_b200 import workload as W  # noqa: E402

sc = W.make_scenario("k1", 200_000, "gtx980", 500, 8, seed=3)
ctx = gd.Context(0)
me = gd.Model.from_forest(sc.energy, ctx)
rows = np.ascontiguousarray(sc.grid.rows)
for n in (10_000, 200_000):
    x = rows[:n]
    me.predict(x)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        me.predict(x)
        ts.append(time.perf_counter() - t0)
    print(f"K1 predict {n} rows x 500 trees d8 (host buffers, incl. copies): {n / min(ts):.3e} rows/s")
try:
    import oracle_lib as O
    t0 = time.perf_counter()
    O.oracle_predict(sc.energy, rows[:2000])
    dt = time.perf_counter() - t0
    print(f"oracle (C restatement, 1 core): {2000 / dt:.3e} rows/s")
except Exception as e:  # noqa: BLE001
    print("oracle timing skipped:", e)
