#!/usr/bin/env python
"""bench.py -- (app x clock) energy+time predictions/s and decisions/s on B200.

One "step" is one pass of the hot path over one batch: the fused sm_100a
kernel evaluates the energy and time GBT ensembles for every (app, clock)
candidate of the batch (rows generated on the fly) and selects one clock per
app (deadline-masked argmin), and -- at N > 1 -- the single NCCL gather of the
per-app decision records.  Default workload = BASELINE.json configs[1]:
10k synthetic apps per GPU x 267 GTX-980-style (sm, mem) clocks, 500-tree
depth-8 energy + time ensembles (weak scaling: every rank owns 10k apps).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c5]
    python bench.py --impl reference ...   # the reference's CPU path

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "(app×freq) energy+time predictions/sec and scheduling decisions/sec at 1/2/4/8 B200"
UNIT = "predictions/s"
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="c2")
    p.add_argument("--cpu-sample-s", type=float, default=10.0, help="target seconds of CPU baseline work")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-clocks", action="store_true", help="skip nvidia-smi sampling (use under ncu)")
    p.add_argument("--w-clk", type=float, default=None, help="experiment: clock-split weight of the synthetic trees")
    p.add_argument("--apps", type=int, default=None, help="override the config's app count (large configs)")
    return p.parse_args()


# configs[3] is quoted as one 10M-app batch row-sharded over 1/2/4/8 GPUs
# (strong scaling); the others fix the apps per GPU (weak scaling).
STRONG = {"c4"}


def workload_config(name: str, world: int, apps=None):
    from paper_2004_08177_b200 import workload as W

    cfg = dict(W.CONFIGS[name])
    if apps:
        cfg["n_apps"] = int(apps)
    if name in STRONG:
        return cfg, -(-cfg["n_apps"] // world), cfg["n_apps"]
    per_rank = cfg["n_apps"]
    return cfg, per_rank, per_rank * world


def deadlines_device(me, mt, ptrs, A, C_, F, K, g, opts, dev, seed):
    """W.deadlines_from_times computed in app chunks on
    the device, so configs[3]'s 10M x 267 time table is never materialised."""
    import torch

    import paper_2004_08177_b200 as gd

    rng = np.random.default_rng(seed)
    q = rng.uniform(0.1, 0.9, size=A)
    bad = rng.random(size=A) < 0.05
    idx = np.minimum((q * (C_ - 1)).astype(np.int64), C_ - 1)
    out = np.empty(A)
    chunk = max(1, min(A, (1 << 28) // (C_ * 8)))
    t_tab = torch.empty((chunk, C_), dtype=torch.float64, device=dev)
    for lo in range(0, A, chunk):
        n = min(chunk, A - lo)
        d = dict(ptrs)
        d["rows"] += lo * F * 8
        d["cat_t"] += lo * K * 8
        d["budgets"] += lo * 8
        d["out"] += lo * 24
        gd.grid_select_device(me, mt, d, n, C_, F, K, g.sm_col, g.mem_col, opts, t_out=t_tab.data_ptr())
        out[lo:lo + n] = deadline_rows(t_tab[:n], idx[lo:lo + n], bad[lo:lo + n])
    return out


def deadline_rows(t_rows, idx, bad):
    """One chunk of W.deadlines_from_times on a (device) tensor of predicted
    times: the idx-th smallest time per app, half the smallest when `bad`."""
    import torch

    srt = torch.sort(t_rows, dim=1).values
    dl = srt.gather(1, torch.from_numpy(idx).to(t_rows.device)[:, None])[:, 0]
    dl = torch.where(torch.from_numpy(bad).to(t_rows.device), srt[:, 0] * 0.5, dl)
    return dl.cpu().numpy()


def make_inputs(cfg, n_total, seed=1234, w_clk=None):
    from paper_2004_08177_b200 import workload as W

    kw = {} if w_clk is None else {"w_clk": w_clk}
    return W.make_scenario("bench", n_total, cfg["catalog"], cfg["n_trees"], cfg["depth"], seed=seed, **kw)


def config_json(name, cfg, per_rank, world, n_clocks):
    return {"workload": f"BASELINE configs[{ {'c2': 1, 'c3': 2, 'c4': 3, 'c5': 4}.get(name, -1) }] ({name}): "
                        f"{per_rank} synthetic apps/GPU x {n_clocks} {cfg['catalog']} clocks, "
                        f"{cfg['n_trees']}-tree depth-{cfg['depth']} GBT energy + time, full_deadline text/energy",
            "apps_per_gpu": per_rank, "apps_total": per_rank * world if name not in STRONG else cfg["n_apps"],
            "clocks": n_clocks,
            "trees_per_model": cfg["n_trees"], "depth": cfg["depth"], "columns": 50,
            "parallelism": f"row-sharded dp{world}",
            "l2": "flushed (512 MiB write) before every timed step", "precision": "exact fp64 (bit-identical)"}


# ---- clocks sampling -----------------------------------------------------------

CLOCK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


class ClockSampler:
    def __init__(self, device: int, path: Path):
        self.path = path
        self.proc = None
        try:
            self.fh = open(path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={CLOCK_FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "samples": len(sm),
                "reasons": sorted(reasons)}


# ---- our arm -------------------------------------------------------------------

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2004_08177_b200 as gd
    from paper_2004_08177_b200 import shard
    from paper_2004_08177_b200 import workload as W

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg, per_rank, n_total = workload_config(args.config, world, args.apps)
    sc = make_inputs(cfg, n_total, w_clk=args.w_clk)
    lo, hi = shard.shard_range(n_total, rank, world)
    A = hi - lo
    g = sc.grid
    C_, F, K = g.n_clocks, g.rows.shape[1], g.cat_t.shape[1]

    ctx = gd.Context(local_rank)
    # One explicit (non-default) stream for everything: torch's flush kernels,
    # the CUDA events and our launches (gd_ctx_set_stream(NULL) would mean
    # "the context's own stream", so the legacy default stream is not used).
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    me = gd.Model.from_forest(sc.energy, ctx)
    mt = gd.Model.from_forest(sc.time, ctx)

    # Device-resident inputs (HBM) for the kernel-timed `value`.
    rows_d = torch.from_numpy(np.ascontiguousarray(g.rows[lo:hi])).to(dev)
    cat_d = torch.from_numpy(np.ascontiguousarray(g.cat_t[lo:hi])).to(dev)
    catc_d = torch.from_numpy(g.cat_cols.astype(np.int32)).to(dev)
    sm_d = torch.from_numpy(g.sm.astype(np.int32)).to(dev)
    mem_d = torch.from_numpy(g.mem.astype(np.int32)).to(dev)
    bud_d = torch.ones(A, dtype=torch.float64, device=dev)
    out_d = torch.zeros(A * shard.DECISION_BYTES, dtype=torch.uint8, device=dev)
    ptrs = dict(rows=rows_d.data_ptr(), cat_t=cat_d.data_ptr(), cat_cols=catc_d.data_ptr(), sm=sm_d.data_ptr(),
                mem=mem_d.data_ptr(), budgets=bud_d.data_ptr(), out=out_d.data_ptr())
    opts = gd.SchedulerOptions(budget="full")

    def launch():
        gd.grid_select_device(me, mt, ptrs, A, C_, F, K, g.sm_col, g.mem_col, opts)

    # Pre-pass (untimed): predicted times -> per-app deadlines.
    budgets = deadlines_device(me, mt, ptrs, A, C_, F, K, g, opts, dev, seed=77 + rank)
    bud_d.copy_(torch.from_numpy(budgets))

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    sampler = None
    if not args.no_clocks:
        out_dir = ROOT / "gpurun_out" if (ROOT / "gpurun_out").is_dir() else Path("/tmp")
        sampler = ClockSampler(local_rank, out_dir / f"clocks_r{rank}.csv")
    try:
        return _timed(args, rank, world, dev, stream, ctx, me, mt, g, sc, cfg, per_rank, n_total, lo, hi, ptrs,
                      out_d, bud_d, budgets, flush, launch, opts, sampler)
    finally:
        if sampler is not None and sampler.proc is not None and sampler.proc.poll() is None:
            sampler.proc.kill()


def _timed(args, rank, world, dev, stream, ctx, me, mt, g, sc, cfg, per_rank, n_total, lo, hi, ptrs, out_d, bud_d,
           budgets, flush, launch, opts, sampler):
    import torch
    import torch.distributed as dist

    import paper_2004_08177_b200 as gd
    from paper_2004_08177_b200 import shard
    from paper_2004_08177_b200 import workload as W

    A = hi - lo
    C_, F, K = g.n_clocks, g.rows.shape[1], g.cat_t.shape[1]

    def step(timing=None):
        flush.zero_()
        if timing is not None:
            timing[0].record(stream)
        launch()
        if timing is not None:
            timing[1].record(stream)
        if world > 1:
            shard.gather_decisions(out_d, n_total, world)
        if timing is not None:
            timing[2].record(stream)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches0 = ctx.launch_count
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    wall0 = time.perf_counter()
    for k in range(args.steps):
        step(evs[k])
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    launches = ctx.launch_count - launches0
    kern_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    step_ms = sum(e[0].elapsed_time(e[2]) for e in evs) / args.steps
    stats = torch.tensor([step_ms, kern_ms, float(launches)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = stats[:2].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = stats[2:].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        stats = torch.cat([mx, tot])
    step_ms, kern_ms, launches = (float(x) for x in stats.cpu())

    # The clock sampler covered the device-timed steps; it stops here so its
    # nvidia-smi queries (every 100 ms, they take the driver lock) cannot land
    # inside the host-API timings below.
    clocks = sampler.stop() if sampler is not None else None

    # e2e: the public host-buffer API (pinned inputs H2D + kernel + D2H decisions).
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    h_grid = W.GridInputs(pin(g.rows[lo:hi]), pin(g.cat_t[lo:hi]), pin(g.cat_cols.astype(np.int32)),
                          pin(g.sm.astype(np.int32)), pin(g.mem.astype(np.int32)), g.sm_col, g.mem_col)
    h_bud = pin(budgets)
    h_out = torch.zeros(A * shard.DECISION_BYTES // 8, dtype=torch.float64).pin_memory().numpy().view(
        gd.DECISION_DTYPE)
    for _ in range(max(args.warmup, 1)):
        gd.grid_select(me, mt, h_grid, h_bud, opts, out=h_out)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e2e_times = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        gd.grid_select(me, mt, h_grid, h_bud, opts, out=h_out)
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = float(np.mean(e2e_times))
    e2e_p50 = float(np.median(e2e_times))
    e2e_max = float(np.max(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # Per-kernel durations (CUDA events recorded by the library around each
    # kernel on the launching stream), in a separate pass so the timed loop
    # above is untouched.
    kern = {}
    ctx.set_timing(True)
    for _ in range(args.steps):
        flush.zero_()
        launch()
        for name, ms in ctx.kernel_times():
            kern.setdefault(name, []).append(ms)
    ctx.set_timing(False)
    kernels_ms = {k: float(np.sum(v) / args.steps) for k, v in kern.items()}
    c5 = c5_latency(me, mt, h_grid, h_bud, opts, A) if rank == 0 else None

    # Consistency: the device-resident run and the e2e run agree.
    dev_dec = out_d.cpu().numpy().view(gd.DECISION_DTYPE)
    consistent = bool(np.array_equal(dev_dec.view(np.uint8), h_out.view(np.uint8)))

    result = None
    if rank == 0:
        dadd_peak = gd.microbench_dadd(ctx)
        units_total = n_total * C_
        value = units_total / (step_ms * 1e-3)
        per_app_bytes = F * 8 + K * 8 + 8 + shard.DECISION_BYTES
        kern_s = kern_ms * 1e-3
        hbm_peak, hbm_src = hbm_peak_gbs()
        achieved_gbs = A * per_app_bytes / kern_s / 1e9
        dom_gbs = A * per_app_bytes / (kernels_ms.get("acc", kern_ms) * 1e-3) / 1e9
        adds = A * C_ * (sc.energy.n_trees + sc.time.n_trees)
        traffic = ncu_traffic(args.config)
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong" if args.config in STRONG else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; models random-init in the reference "
                                                           "GbtNode format, rows in the reference 50-column schema)",
            "config": config_json(args.config, cfg, per_rank, world, C_),
            "decisions_per_s": n_total / (step_ms * 1e-3),
            "kernel_ms": kern_ms,
            "roofline": {"bound": "hbm", "kernel": "grid_acc_kernel (dominant)", "achieved": dom_gbs,
                         "peak": hbm_peak, "unit": "GB/s", "frac": dom_gbs / hbm_peak, "traffic": traffic,
                         "peak_source": hbm_src,
                         "algorithmic_bytes_per_app": per_app_bytes,
                         "achieved_whole_step": achieved_gbs,
                         "note": "HBM is not the binding resource (SURVEY 8d): compulsory bytes are "
                                 f"{per_app_bytes} B per app = {per_app_bytes / C_:.2f} B per prediction; "
                                 "traffic = ncu dram read+write bytes of one grid_acc_kernel launch "
                                 "(profiles/ncu_traffic.json)"},
            "kernels_ms": kernels_ms,
            "binding_roofline": {"bound": "fp64_ordered_add", "kernel": "grid_acc_kernel (dominant)",
                                 "achieved": adds / (kernels_ms.get("acc", kern_ms) * 1e-3), "peak": dadd_peak,
                                 "unit": "adds/s", "frac": adds / (kernels_ms.get("acc", kern_ms) * 1e-3) / dadd_peak,
                                 "frac_whole_step": adds / kern_s / dadd_peak,
                                 "adds_per_prediction": sc.energy.n_trees + sc.time.n_trees,
                                 "peak_source": "measured in-run (gd_microbench_dadd, 8 independent __dadd_rn "
                                                "chains/thread)"},
            "e2e": {"value": units_total / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": int(A * (F + K + 1) * 8 + K * 4 + C_ * 8),
                    "d2h_bytes_per_step": int(A * shard.DECISION_BYTES), "ms_per_step": e2e_s * 1e3,
                    "ms_p50": e2e_p50 * 1e3, "ms_max": e2e_max * 1e3,
                    "api": "gd_grid_select (C ABI, pinned host buffers)"},
            "gpu_launches": int(launches),
            "wall_ms_per_step_incl_l2_flush": wall / args.steps * 1e3,
            "clocks": clocks, "device_vs_e2e_decisions_identical": consistent,
            "c5_latency": c5,
        }
        if world == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"] = cpu_baseline(sc, budgets, args.cpu_sample_s, dev_dec)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


def c5_latency(me, mt, h_grid, h_bud, opts, A, batch=64, iters=300, warmup=30):
    """BASELINE configs[4]: the online scheduler stream -- 64-job arrival
    batches x the same 267-clock catalog and 500-tree models, each batch one
    gd_grid_select call on pinned host buffers (H2D, kernels, D2H inside the
    wall-clock latency).  Successive batches take successive 64-app windows."""
    import paper_2004_08177_b200 as gd
    from paper_2004_08177_b200 import workload as W

    g = h_grid
    n_win = max(1, A // batch)
    wins = []
    for w in range(min(n_win, 64)):
        lo = w * batch
        wins.append((W.GridInputs(g.rows[lo:lo + batch], g.cat_t[lo:lo + batch], g.cat_cols, g.sm, g.mem, g.sm_col,
                                  g.mem_col), np.ascontiguousarray(h_bud[lo:lo + batch])))
    out = np.zeros(batch, gd.DECISION_DTYPE)
    lat = []
    for k in range(warmup + iters):
        gw, bw = wins[k % len(wins)]
        t0 = time.perf_counter()
        gd.grid_select(me, mt, gw, bw, opts, out=out)
        if k >= warmup:
            lat.append(time.perf_counter() - t0)
    lat_us = np.array(lat) * 1e6
    return {"workload": "BASELINE configs[4] (c5): 64-job batches x 267 clocks, 500-tree depth-8 E + T, one "
                        "gd_grid_select per batch (host buffers)",
            "p50_us": float(np.percentile(lat_us, 50)), "p99_us": float(np.percentile(lat_us, 99)),
            "mean_us": float(lat_us.mean()), "batches": iters,
            "decisions_per_s_at_p50": batch / (np.percentile(lat_us, 50) * 1e-6),
            "predictions_per_s_at_p50": batch * g.n_clocks / (np.percentile(lat_us, 50) * 1e-6)}


def hbm_peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except (KeyError, ValueError):
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(config)
        except ValueError:
            return None
    return None


def cpu_baseline(sc, budgets, target_s, gpu_dec):
    """The reference's own predict + schedule_d_dvfs (oracle/_ref, compiled from
    the reference sources) on 1 host thread over a bounded app sample."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O

    g = sc.grid
    if O.ref_available():
        n = 4
        secs, _ = O.ref_bench_grid(sc.energy, sc.time, g, budgets, n, 1)
        n = int(max(4, min(g.n_apps, target_s / max(secs / n, 1e-6))))
        secs, dec = O.ref_bench_grid(sc.energy, sc.time, g, budgets, n, 1)
        kind = "reference"
    else:
        sub_n = 4
        t0 = time.perf_counter()
        O.oracle_grid(sc.energy, sc.time, g, budgets, app_slice=(0, sub_n))
        per = (time.perf_counter() - t0) / sub_n
        n = int(max(4, min(g.n_apps, target_s / max(per, 1e-6))))
        t0 = time.perf_counter()
        dec, _, _ = O.oracle_grid(sc.energy, sc.time, g, budgets, app_slice=(0, n))
        secs = time.perf_counter() - t0
        kind = "port"
    match = bool(np.array_equal(dec.view(np.uint8), gpu_dec[:n].view(np.uint8)))
    return {"value": n * g.n_clocks / secs, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"first {n} apps x {g.n_clocks} clocks ({n * g.n_clocks} predictions) of the same workload, "
                      f"materialised rows -> models::predict (E, T) -> schedule_d_dvfs(full_deadline); {secs:.1f} s",
            "decisions_match_gpu": match}


# ---- reference arm -------------------------------------------------------------

def run_reference(args, rank, world):
    if rank != 0:
        return None
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O

    cfg, per_rank, n_total = workload_config(args.config, world, args.apps)
    if not O.ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libgpudvfs_ref.so not built"}
    sc = make_inputs(cfg, min(n_total, 4096))
    g = sc.grid
    threads = os.cpu_count() or 1
    # deadlines from the reference's own predicted times on the sample (untimed)
    budgets = np.ones(g.n_apps)
    n_probe = threads * 2
    secs, _ = O.ref_bench_grid(sc.energy, sc.time, g, budgets, n_probe, threads)
    per_step_target = max(1.0, min(6.0, 150.0 / max(args.steps + args.warmup, 1)))
    n = int(max(threads, min(g.n_apps, per_step_target / max(secs / n_probe, 1e-9))))
    for _ in range(max(args.warmup, 0)):
        O.ref_bench_grid(sc.energy, sc.time, g, budgets, n, threads)
    times = []
    for _ in range(args.steps):
        s, _ = O.ref_bench_grid(sc.energy, sc.time, g, budgets, n, threads)
        times.append(s)
    step_s = float(np.mean(times))
    value = n * g.n_clocks / step_s
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.config in STRONG else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_json(args.config, cfg, per_rank, world, g.n_clocks),
        "decisions_per_s": n / step_s,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{n} apps x {g.n_clocks} clocks per step, {threads} threads on contiguous app "
                                   "partitions: materialised rows -> models::predict (E, T) -> "
                                   "schedule_d_dvfs(full_deadline)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if "RANK" in os.environ else 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, world, local_rank)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
