"""configs[4] latency probe: the 64-job stream as in bench.py's c5_latency
(L2 warm, no flush), with per-interval device times from the timing hook
(h2d | rank | walk | acc | d2h) and the wall latency."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2004_08177_b200 as gd  # noqa: E402
from paper_2004_08177_b200 import workload as W  # noqa: E402

A, B = 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 64
sc = W.make_scenario("c5", A, "gtx980", 500, 8, seed=1234)
ctx = gd.Context(0)
me, mt = gd.Model.from_forest(sc.energy, ctx), gd.Model.from_forest(sc.time, ctx)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
g = sc.grid
opts = gd.SchedulerOptions(budget="full")
wins = [(W.GridInputs(pin(g.rows[lo:lo + B]), pin(g.cat_t[lo:lo + B]), pin(g.cat_cols.astype(np.int32)), pin(g.sm),
                      pin(g.mem), g.sm_col, g.mem_col), pin(np.ones(B))) for lo in range(0, A - B + 1, B)][:64]
out = pin(np.zeros(B, gd.DECISION_DTYPE).view(np.uint8)).view(gd.DECISION_DTYPE)
lat = []
for k in range(330):
    gw, bw = wins[k % len(wins)]
    t0 = time.perf_counter()
    gd.grid_select(me, mt, gw, bw, opts, out=out)
    if k >= 30:
        lat.append(time.perf_counter() - t0)
lat = np.array(lat) * 1e6
ctx.set_timing(True)
spans = []
for k in range(100):
    gw, bw = wins[k % len(wins)]
    gd.grid_select(me, mt, gw, bw, opts, out=out)
    spans.append(dict(ctx.kernel_times()))
ctx.set_timing(False)
med = {k: round(float(np.median([s.get(k, 0) for s in spans])) * 1e3, 1) for k in spans[0]}
print(f"B={B}: wall p50 {np.percentile(lat, 50):.1f} us p99 {np.percentile(lat, 99):.1f} us | timed intervals (us) {med} "
      f"sum {sum(med.values()):.1f}")

# Device-resident inputs: CPU enqueue cost of one grid_select_device call,
# the synchronous device latency, and the pipelined per-call time.
dev = torch.device("cuda")
gw, bw = wins[0]
keep = dict(rows=torch.from_numpy(gw.rows).to(dev), cat_t=torch.from_numpy(gw.cat_t).to(dev),
            cat_cols=torch.from_numpy(gw.cat_cols).to(dev), sm=torch.from_numpy(gw.sm.astype(np.int32)).to(dev),
            mem=torch.from_numpy(gw.mem.astype(np.int32)).to(dev), budgets=torch.from_numpy(bw).to(dev),
            out=torch.zeros(B * 32, dtype=torch.uint8, device=dev))
ptrs = {k: v.data_ptr() for k, v in keep.items()}
C_, F, K = g.n_clocks, g.rows.shape[1], g.cat_t.shape[1]
ctx.set_stream(torch.cuda.current_stream().cuda_stream)


def dev_call():
    gd.grid_select_device(me, mt, ptrs, B, C_, F, K, g.sm_col, g.mem_col, opts)


for _ in range(20):
    dev_call()
torch.cuda.synchronize()
enq, syn = [], []
for _ in range(200):
    t0 = time.perf_counter()
    dev_call()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    enq.append(t1 - t0)
    syn.append(t2 - t0)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    dev_call()
torch.cuda.synchronize()
pipe = (time.perf_counter() - t0) / 200
print(f"B={B} device-resident: enqueue p50 {1e6 * np.median(enq):.1f} us | enqueue+sync p50 {1e6 * np.median(syn):.1f} us"
      f" | pipelined {1e6 * pipe:.1f} us/call")

# Python wrapper overhead vs the bare C call (same prebuilt arguments).
import ctypes as Ct  # noqa: E402
from paper_2004_08177_b200 import _capi  # noqa: E402
gs = _capi.Grid(ptrs["rows"], B, F, K, ptrs["cat_t"], ptrs["cat_cols"], None, B, ptrs["sm"], ptrs["mem"], C_,
                g.sm_col, g.mem_col, 0, ptrs["budgets"])
op = opts.opts()
fn = _capi.lib().gd_grid_select_device
args = (ctx.handle, me.handle, mt.handle, Ct.byref(gs), Ct.byref(op), ptrs["out"], None, None)
torch.cuda.synchronize()
bare = []
for _ in range(200):
    t0 = time.perf_counter()
    fn(*args)
    bare.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
print(f"B={B} bare C enqueue p50 {1e6 * np.median(bare):.1f} us")
