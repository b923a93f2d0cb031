#!/usr/bin/env python
"""bench.py -- (app x clock) energy+time predictions/s and decisions/s on B200.

One "step" is one pass of the hot path over the whole batch: for every
(app, clock) candidate the energy and time GBT ensembles are evaluated
(candidate rows generated on the fly inside the kernels), one clock is
selected per app (deadline-masked argmin, full_deadline budgets), and -- at
N > 1 -- the single NCCL gather of the 24-byte per-app decision records to
rank 0.

Default workload = BASELINE.json configs[3], the config the metric is quoted
on ("at 1/2/4/8 B200"): 10,000,000 synthetic apps x 267 GTX-980-style
(sm, mem) clocks, 2000-tree depth-12 energy + time ensembles, one batch
row-sharded over the N GPUs (strong scaling).  configs[2] (1M x 200,
1000-tree depth-10), configs[1] (10k x 267, 500-tree depth-8) and the
configs[4] latency stream are measured in the same run as extra keys.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c3|c2]
    python bench.py --impl reference ...   # the reference's CPU path

--gpus N > 1 without torchrun env re-executes itself under
``torch.distributed.run`` (one rank per GPU, 127.0.0.1 rendezvous).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
CFG_INDEX = {"c2": 1, "c2t": 1, "c3": 2, "c4": 3, "c5": 4}
DEADLINE_SEED = 77


def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="c4")
    p.add_argument("--cpu-sample-s", type=float, default=10.0, help="target seconds of CPU baseline work")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip the configs[1]/[2]/[4] extra keys")
    p.add_argument("--no-clocks", action="store_true", help="skip nvidia-smi sampling (use under ncu)")
    p.add_argument("--e2e-steps", type=int, default=3, help="host-API (e2e) steps, capped at --steps")
    p.add_argument("--w-clk", type=float, default=None, help="experiment: clock-split weight of the synthetic trees")
    p.add_argument("--apps", type=int, default=None, help="override the config's app count")
    return p.parse_args(argv)


# configs[3] is quoted as one 10M-app batch row-sharded over 1/2/4/8 GPUs
# (strong scaling); the others fix the apps per GPU (weak scaling).
STRONG = {"c4"}


def workload_config(name: str, world: int, apps=None):
    """(config, apps per rank (max), apps in the whole job)."""
    from paper_2004_08177_b200 import workload as W

    cfg = dict(W.CONFIGS[name])
    if apps:
        cfg["n_apps"] = int(apps)
    if name in STRONG:
        return cfg, -(-cfg["n_apps"] // world), cfg["n_apps"]
    per_rank = cfg["n_apps"]
    return cfg, per_rank, per_rank * world


def make_inputs(cfg, n_total, app_range, seed=1234, w_clk=None):
    """The config's scenario, built for global apps [lo, hi) only (rows are
    chunk-seeded: every rank's shard and the reference arm's sample are
    slices of one n_total-app batch)."""
    from paper_2004_08177_b200 import workload as W

    if cfg.get("trained"):
        return W.make_trained_scenario("bench", n_total, cfg["catalog"], cfg["n_trees"], cfg["depth"], seed=seed,
                                       app_range=app_range)
    kw = {} if w_clk is None else {"w_clk": w_clk}
    return W.make_scenario("bench", n_total, cfg["catalog"], cfg["n_trees"], cfg["depth"], seed=seed,
                           chunked=True, app_range=app_range, **kw)


def deadline_rows(t_rows, idx, bad):
    """One chunk of the deadlines_from_times rule on a (device) tensor of
    predicted times: the idx-th smallest time per app, half the smallest
    when `bad`."""
    import torch

    srt = torch.sort(t_rows, dim=1).values
    dl = srt.gather(1, torch.from_numpy(idx).to(t_rows.device)[:, None])[:, 0]
    dl = torch.where(torch.from_numpy(bad).to(t_rows.device), srt[:, 0] * 0.5, dl)
    return dl.cpu().numpy()


def deadlines_device(me, mt, ptrs, A, C_, F, K, g, opts, dev, lo):
    """Per-app deadlines (a seeded quantile of the app's
    own predicted times) for global apps [lo, lo + A), computed in app chunks
    on the device so configs[3]'s 10M x 267 time table is never
    materialised.  Draws are chunk-seeded by global app index
    (workload.deadline_draws), so the reference arm reproduces them."""
    import torch

    import paper_2004_08177_b200 as gd
    from paper_2004_08177_b200 import workload as W

    q, bad = W.deadline_draws(DEADLINE_SEED, lo, lo + A)
    idx = np.minimum((q * (C_ - 1)).astype(np.int64), C_ - 1)
    out = np.empty(A)
    chunk = max(1, min(A, (1 << 28) // (C_ * 8)))
    t_tab = torch.empty((chunk, C_), dtype=torch.float64, device=dev)
    for a in range(0, A, chunk):
        n = min(chunk, A - a)
        d = dict(ptrs)
        d["rows"] += a * F * 8
        d["cat_t"] += a * K * 8
        d["budgets"] += a * 8
        d["out"] += a * 24
        gd.grid_select_device(me, mt, d, n, C_, F, K, g.sm_col, g.mem_col, opts, t_out=t_tab.data_ptr())
        out[a:a + n] = deadline_rows(t_tab[:n], idx[a:a + n], bad[a:a + n])
    return out


def config_json(name, cfg, per_rank, n_total, world, n_clocks):
    return {"workload": f"BASELINE configs[{CFG_INDEX.get(name, -1)}] ({name}): {n_total} synthetic apps "
                        f"({'one batch row-sharded over' if name in STRONG else 'fixed per GPU on'} {world} GPU"
                        f"{'s' if world > 1 else ''}) x {n_clocks} {cfg['catalog']} clocks, {cfg['n_trees']}-tree "
                        f"depth-{cfg['depth']} GBT energy + time"
                        f"{' TRAINED on profiled records (GPU fit_gbt)' if cfg.get('trained') else ''}"
                        f", full_deadline text/energy",
            "apps_per_gpu": per_rank, "apps_total": n_total, "clocks": n_clocks,
            "trees_per_model": cfg["n_trees"], "depth": cfg["depth"], "columns": 50,
            "parallelism": f"row-sharded dp{world}",
            "l2": "flushed (512 MiB write) before every timed step; inputs "
                  f"{'> L2' if per_rank * 448 > (126 << 20) else '< L2'}",
            "precision": "exact fp64 (bit-identical)"}


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

class Arm:
    """One rank's share of one config: models, device-resident inputs, the
    deadline pre-pass, and the step."""

    def __init__(self, name, rank, world, dev, ctx, stream, apps=None, w_clk=None):
        import torch

        import paper_2004_08177_b200 as gd
        from paper_2004_08177_b200 import shard

        self.name, self.rank, self.world, self.dev, self.ctx = name, rank, world, dev, ctx
        self.cfg, self.per_rank, self.n_total = workload_config(name, world, apps)
        self.lo, self.hi = shard.shard_range(self.n_total, rank, world)
        self.A = self.hi - self.lo
        sc = make_inputs(self.cfg, self.n_total, (self.lo, self.hi), w_clk=w_clk)
        self.sc = sc
        g = self.g = sc.grid
        self.C, self.F, self.K = g.n_clocks, g.rows.shape[1], g.cat_t.shape[1]
        self.me = gd.Model.from_forest(sc.energy, ctx)
        self.mt = gd.Model.from_forest(sc.time, ctx)
        self.rows_d = torch.from_numpy(g.rows).to(dev)
        self.cat_d = torch.from_numpy(g.cat_t).to(dev)
        self.catc_d = torch.from_numpy(g.cat_cols.astype(np.int32)).to(dev)
        self.sm_d = torch.from_numpy(g.sm.astype(np.int32)).to(dev)
        self.mem_d = torch.from_numpy(g.mem.astype(np.int32)).to(dev)
        self.bud_d = torch.ones(self.A, dtype=torch.float64, device=dev)
        self.out_d = torch.zeros(self.A * shard.DECISION_BYTES, dtype=torch.uint8, device=dev)
        self.ptrs = dict(rows=self.rows_d.data_ptr(), cat_t=self.cat_d.data_ptr(), cat_cols=self.catc_d.data_ptr(),
                         sm=self.sm_d.data_ptr(), mem=self.mem_d.data_ptr(), budgets=self.bud_d.data_ptr(),
                         out=self.out_d.data_ptr())
        self.opts = gd.SchedulerOptions(budget="full")
        # Pre-pass (untimed): predicted times -> per-app deadlines.
        self.budgets = deadlines_device(self.me, self.mt, self.ptrs, self.A, self.C, self.F, self.K, g, self.opts,
                                        dev, self.lo)
        self.bud_d.copy_(torch.from_numpy(self.budgets))
        torch.cuda.synchronize(dev)

    def attach_comm(self, comm):
        """The decision gather of N > 1 ranks (gd_comm, one NCCL gather to rank 0)."""
        import torch

        from paper_2004_08177_b200 import shard

        self.comm = comm
        self.counts = [hi - lo for lo, hi in (shard.shard_range(self.n_total, r, self.world) for r in range(self.world))]
        self.recv_d = (torch.empty(self.n_total * shard.DECISION_BYTES, dtype=torch.uint8, device=self.dev)
                       if comm is not None and self.rank == 0 else None)

    def gather(self):
        """Enqueue the gather on the context stream; rank 0 gets every app's decision (recv_d)."""
        self.comm.gather_decisions(self.out_d.data_ptr(), self.counts,
                                   self.recv_d.data_ptr() if self.recv_d is not None else 0, 0)
        return self.recv_d

    def launch(self):
        import paper_2004_08177_b200 as gd

        gd.grid_select_device(self.me, self.mt, self.ptrs, self.A, self.C, self.F, self.K, self.g.sm_col,
                              self.g.mem_col, self.opts)

    @property
    def units(self):
        return self.n_total * self.C

    def adds(self):
        return self.A * self.C * (self.sc.energy.n_trees + self.sc.time.n_trees)

    def per_app_bytes(self):
        from paper_2004_08177_b200 import shard

        return self.F * 8 + self.K * 8 + 8 + shard.DECISION_BYTES


def _barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _max_over_ranks(vals, world, dev):
    import torch
    import torch.distributed as dist

    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2004_08177_b200 as gd

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ctx = gd.Context(local_rank)
    comm = None
    if world > 1:
        # The decision gather runs through the library's own NCCL
        # communicator (gd_comm): rank 0 makes the id, torch.distributed
        # only carries it.
        box = [gd.Comm.make_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        comm = gd.Comm(ctx, box[0], world, rank)
    # One explicit (non-default) stream for everything: torch's flush kernels,
    # the CUDA events and our launches.
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    t_setup = time.perf_counter()
    arm = Arm(args.config, rank, world, dev, ctx, stream, args.apps, args.w_clk)
    arm.attach_comm(comm)
    setup_s = time.perf_counter() - t_setup
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    sampler = None
    if not args.no_clocks:
        out_dir = ROOT / "gpurun_out" if (ROOT / "gpurun_out").is_dir() else Path("/tmp")
        sampler = ClockSampler(local_rank, out_dir / f"clocks_r{rank}.csv")
    try:
        res = timed_main(args, arm, rank, world, dev, stream, ctx, flush, sampler)
    finally:
        if sampler is not None and sampler.proc is not None and sampler.proc.poll() is None:
            sampler.proc.kill()
    if rank == 0 and res is not None:
        res["setup_s"] = setup_s
        if world == 1 and not args.no_extras:
            res["extra_configs"] = extras(args, arm, dev, ctx, stream, flush)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return res


def device_steps(arm, steps, warmup, world, stream, flush, gather=True):
    """W untimed + K timed steps; returns (step ms, kernel ms), max over ranks."""
    import torch

    from paper_2004_08177_b200 import shard

    def step(ev=None):
        flush.zero_()
        if ev is not None:
            ev[0].record(stream)
        arm.launch()
        if ev is not None:
            ev[1].record(stream)
        if world > 1 and gather:
            arm.gather()
        if ev is not None:
            ev[2].record(stream)

    for _ in range(max(warmup, 0)):
        step()
    torch.cuda.synchronize(arm.dev)
    _barrier(world)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    torch.cuda.synchronize(arm.dev)
    _barrier(world)
    for k in range(steps):
        step(evs[k])
    torch.cuda.synchronize(arm.dev)
    _barrier(world)
    kern_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / steps
    step_ms = sum(e[0].elapsed_time(e[2]) for e in evs) / steps
    return _max_over_ranks([step_ms, kern_ms], world, arm.dev)


def timed_main(args, arm, rank, world, dev, stream, ctx, flush, sampler):
    import torch
    import torch.distributed as dist

    import paper_2004_08177_b200 as gd
    from paper_2004_08177_b200 import shard
    from paper_2004_08177_b200 import workload as W

    launches0 = ctx.launch_count
    wall0 = time.perf_counter()
    step_ms, kern_ms = device_steps(arm, args.steps, args.warmup, world, stream, flush)
    wall = time.perf_counter() - wall0
    launches = ctx.launch_count - launches0
    tot = torch.tensor([float(launches)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    launches = float(tot.item()) * args.steps / max(args.steps + args.warmup, 1)
    # The clock sampler covered the device-timed steps; it stops here so its
    # nvidia-smi queries (they take the driver lock) cannot land inside the
    # host-API timings below.
    clocks = sampler.stop() if sampler is not None else None

    # e2e through the public API with HOST buffers: the host->device copy of
    # the step's inputs and the device->host read of its decisions inside the
    # timed region.  N = 1: gd_grid_select (C ABI, pinned host buffers).  N > 1:
    # each rank copies its shard in, runs the device entry, the decisions are
    # gathered to rank 0 over NCCL and read back there.
    g = arm.g
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    e2e_steps = max(1, min(args.e2e_steps, args.steps))
    e2e_times = []
    if world == 1:
        h_grid = W.GridInputs(pin(g.rows).numpy(), pin(g.cat_t).numpy(), pin(g.cat_cols.astype(np.int32)).numpy(),
                              pin(g.sm.astype(np.int32)).numpy(), pin(g.mem.astype(np.int32)).numpy(), g.sm_col,
                              g.mem_col)
        h_bud = pin(arm.budgets).numpy()
        h_out = torch.zeros(arm.A * shard.DECISION_BYTES // 8, dtype=torch.float64).pin_memory().numpy().view(
            gd.DECISION_DTYPE)
        gd.grid_select(arm.me, arm.mt, h_grid, h_bud, arm.opts, out=h_out)
        for _ in range(e2e_steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            gd.grid_select(arm.me, arm.mt, h_grid, h_bud, arm.opts, out=h_out)
            e2e_times.append(time.perf_counter() - t0)
        h2d = int(arm.A * (arm.F + arm.K + 1) * 8 + arm.K * 4 + arm.C * 8)
        d2h = int(arm.A * shard.DECISION_BYTES)
        api = "gd_grid_select (C ABI, pinned host buffers)"
        host_dec = h_out
    else:
        h_rows, h_cat, h_bud = pin(g.rows), pin(g.cat_t), pin(arm.budgets)
        full_h = torch.empty(arm.n_total * shard.DECISION_BYTES, dtype=torch.uint8).pin_memory()

        def e2e_step():
            arm.rows_d.copy_(h_rows, non_blocking=True)
            arm.cat_d.copy_(h_cat, non_blocking=True)
            arm.bud_d.copy_(h_bud, non_blocking=True)
            arm.launch()
            full = arm.gather()
            if rank == 0:
                full_h.copy_(full, non_blocking=True)
            torch.cuda.synchronize(dev)

        e2e_step()
        for _ in range(e2e_steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            _barrier(world)
            t0 = time.perf_counter()
            e2e_step()
            _barrier(world)
            e2e_times.append(time.perf_counter() - t0)
        h2d = int(arm.A * (arm.F + arm.K + 1) * 8)
        d2h = int(arm.n_total * shard.DECISION_BYTES) if rank == 0 else 0
        api = "grid_select_device on each rank's shard (H2D from pinned host) + gd_gather_decisions (NCCL gather to rank 0) + D2H"
        host_dec = full_h.numpy()[: arm.A * shard.DECISION_BYTES].view(gd.DECISION_DTYPE) if rank == 0 else None
    e2e_s, e2e_max = _max_over_ranks([float(np.mean(e2e_times)), float(np.max(e2e_times))], world, dev)

    # Per-kernel durations (CUDA events recorded by the library around each
    # kernel on the launching stream), one extra step so the timed loop above
    # is untouched.
    kern = {}
    ctx.set_timing(True)
    flush.zero_()
    arm.launch()
    for name, ms in ctx.kernel_times():
        kern[name] = kern.get(name, 0.0) + ms
    ctx.set_timing(False)
    torch.cuda.synchronize(dev)

    # Consistency: the device-resident run and the e2e run agree.
    dev_dec = arm.out_d.cpu().numpy().view(gd.DECISION_DTYPE)
    consistent = None if host_dec is None else bool(np.array_equal(dev_dec.view(np.uint8),
                                                                   host_dec.view(np.uint8)))
    if rank != 0:
        return None
    dadd_peak = gd.microbench_dadd(ctx)
    value = arm.units / (step_ms * 1e-3)
    kern_s = kern_ms * 1e-3
    hbm_peak, hbm_src = hbm_peak_gbs()
    acc_ms = kern.get("acc", kern_ms)
    achieved_gbs = arm.A * arm.per_app_bytes() / kern_s / 1e9
    dom_gbs = arm.A * arm.per_app_bytes() / (acc_ms * 1e-3) / 1e9
    adds = arm.adds()
    traffic = ncu_traffic(arm.name)
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong" if arm.name in STRONG else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, chunk-seeded rows; models random-init in the reference GbtNode format, rows in "
                "the reference 50-column schema)",
        "config": config_json(arm.name, arm.cfg, arm.per_rank, arm.n_total, world, arm.C),
        "decisions_per_s": arm.n_total / (step_ms * 1e-3),
        "kernel_ms": kern_ms,
        "roofline": {"bound": "hbm", "kernel": "grid_acc_kernel (dominant)", "achieved": dom_gbs,
                     "peak": hbm_peak, "unit": "GB/s", "frac": dom_gbs / hbm_peak, "traffic": traffic,
                     "peak_source": hbm_src, "algorithmic_bytes_per_app": arm.per_app_bytes(),
                     "achieved_whole_step": achieved_gbs,
                     "note": "HBM is not the binding resource (SURVEY 8d): compulsory bytes are "
                             f"{arm.per_app_bytes()} B per app = {arm.per_app_bytes() / arm.C:.2f} B per prediction; "
                             "traffic = ncu dram read+write bytes of the dominant kernel per launch "
                             "(profiles/ncu_traffic.json); see binding_roofline"},
        "kernels_ms": kern,
        "binding_roofline": {"bound": "fp64_ordered_add", "kernel": "grid_acc_kernel (dominant)",
                             "achieved": adds / (acc_ms * 1e-3), "peak": dadd_peak, "unit": "adds/s",
                             "frac": adds / (acc_ms * 1e-3) / dadd_peak,
                             "frac_whole_step": adds / kern_s / dadd_peak,
                             "adds_per_prediction": arm.sc.energy.n_trees + arm.sc.time.n_trees,
                             "formula": "apps x clocks x (T_e + T_t) in-order __dadd_rn / kernel time",
                             "peak_source": "measured in-run (gd_microbench_dadd, 8 independent __dadd_rn "
                                            "chains/thread)"},
        "e2e": {"value": arm.units / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1e3, "ms_max": e2e_max * 1e3, "steps": e2e_steps, "api": api},
        "gpu_launches": int(round(launches)),
        "wall_ms_per_step_incl_l2_flush": wall / max(args.steps + args.warmup, 1) * 1e3,
        "clocks": clocks, "device_vs_e2e_decisions_identical": consistent,
    }
    if world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(arm, args.cpu_sample_s, dev_dec)
    return result


def extras(args, main_arm, dev, ctx, stream, flush):
    """configs[1] / configs[2] (short device-timed runs) and the configs[4]
    latency stream, beside the headline (N = 1)."""
    import torch

    from paper_2004_08177_b200 import workload as W

    out = {}
    for name in ("c3", "c2", "c2t"):
        if name == main_arm.name:
            continue
        try:
            arm = Arm(name, 0, 1, dev, ctx, stream)
            steps = 3 if name == "c3" else 10
            step_ms, kern_ms = device_steps(arm, steps, 3, 1, stream, flush)
            kern = {}
            ctx.set_timing(True)
            flush.zero_()
            arm.launch()
            for k, ms in ctx.kernel_times():
                kern[k] = kern.get(k, 0.0) + ms
            ctx.set_timing(False)
            dadd = arm.adds() / (kern.get("acc", kern_ms) * 1e-3)
            out[name] = {"config": config_json(name, arm.cfg, arm.per_rank, arm.n_total, 1, arm.C),
                         "value": arm.units / (step_ms * 1e-3), "unit": UNIT, "ms_per_step": step_ms,
                         "steps": steps, "warmup": 3, "kernels_ms": kern,
                         "acc_fp64_add_rate": dadd,
                         "decisions_per_s": arm.n_total / (step_ms * 1e-3)}
            if name in ("c2", "c2t"):
                # walk-record mix (CPU analysis of the first 48 apps): random
                # synthetic trees vs trees trained on profiled records
                out[name]["record_kinds"] = {
                    m: W.record_kinds(f, arm.g.rows, arm.g.sm_col, arm.g.mem_col, max_apps=48)
                    for m, f in (("energy", arm.sc.energy), ("time", arm.sc.time))}
            if name == "c2":
                out["c5_latency"] = c5_latency(arm)
            del arm
            torch.cuda.empty_cache()
        except Exception as e:  # an extra must not cost the headline line
            out[name] = {"error": repr(e)}
    try:
        c1 = run_c1(argparse.Namespace(apps=100, steps=9), "ours")
        out["c1"] = {k: c1[k] for k in ("config", "value", "unit", "ms_per_step", "decisions_per_s", "cpu_baseline",
                                        "decisions_identical_to_reference")}
        # An untimed pass first: the first 1250-job process on a fresh box ran
        # with a 2.5x slower median (host warm-up), the next ones did not.
        run_c1(argparse.Namespace(apps=1000, steps=1), "ours")
        c1k = run_c1(argparse.Namespace(apps=1000, steps=9), "ours")
        out["c1_1000_jobs"] = {k: c1k[k] for k in ("value", "ms_per_step", "decisions_per_s", "cpu_baseline",
                                                   "decisions_identical_to_reference")}
    except Exception as e:  # noqa: BLE001
        out["c1"] = {"error": repr(e)}
    return out


def c5_latency(arm, batch=64, iters=300, warmup=30):
    """BASELINE configs[4]: the online scheduler stream -- 64-job arrival
    batches x the 267-clock catalog and configs[1]'s 500-tree models, each
    batch one gd_grid_select call on host buffers (H2D, kernels, D2H inside
    the wall-clock latency).  Successive batches take successive 64-app
    windows."""
    import paper_2004_08177_b200 as gd
    from paper_2004_08177_b200 import workload as W

    g = arm.g
    n_win = max(1, arm.A // batch)
    wins = []
    for w in range(min(n_win, 64)):
        lo = w * batch
        wins.append((W.GridInputs(np.ascontiguousarray(g.rows[lo:lo + batch]),
                                  np.ascontiguousarray(g.cat_t[lo:lo + batch]), g.cat_cols.astype(np.int32),
                                  g.sm.astype(np.int32), g.mem.astype(np.int32), g.sm_col, g.mem_col),
                     np.ascontiguousarray(arm.budgets[lo:lo + batch])))
    out = np.zeros(batch, gd.DECISION_DTYPE)
    lat = []
    for k in range(warmup + iters):
        gw, bw = wins[k % len(wins)]
        t0 = time.perf_counter()
        gd.grid_select(arm.me, arm.mt, gw, bw, arm.opts, out=out)
        if k >= warmup:
            lat.append(time.perf_counter() - t0)
    lat_us = np.array(lat) * 1e6
    # CPU baseline of the same stream: the reference's predict + select per
    # batch (oracle/_ref) on all host threads, 40 batches.
    cpu = None
    try:
        sys.path.insert(0, str(ROOT / "tests"))
        import oracle_lib as O

        if O.ref_available():
            threads = os.cpu_count() or 1
            cl = []
            for k in range(40):
                gw, bw = wins[k % len(wins)]
                secs, _ = O.ref_bench_grid(arm.sc.energy, arm.sc.time, gw, bw, batch, threads)
                cl.append(secs * 1e6)
            cl = np.array(cl)
            cpu = {"kind": "reference", "cores": threads, "batches": 40, "p50_us": float(np.percentile(cl, 50)),
                   "p99_us": float(np.percentile(cl, 99))}
    except Exception as e:  # noqa: BLE001
        cpu = {"error": repr(e)}
    return {"workload": "BASELINE configs[4] (c5): 64-job batches x 267 clocks, 500-tree depth-8 E + T, one "
                        "gd_grid_select per batch (host buffers)",
            "cpu_reference": cpu,
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


# ---- CPU legs (the checker: oracle/_ref, or the oracle port) --------------------

def cpu_sample_grid(cfg, n_total, n, w_clk=None):
    """The first n apps of the same n_total-app batch, with the deadlines our
    arm uses for them (draws by global app index; times from the CPU path
    itself, untimed)."""
    from paper_2004_08177_b200 import workload as W

    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O

    sc = make_inputs(cfg, n_total, (0, n), w_clk=w_clk)
    g = sc.grid
    if O.ref_available():
        _, _, t = O.ref_grid_tables(sc.energy, sc.time, g)
    else:
        _, _, t = O.oracle_grid(sc.energy, sc.time, g, np.ones(n))
    q, bad = W.deadline_draws(DEADLINE_SEED, 0, n)
    return sc, W.deadlines_from_draws(t, q, bad)


def cpu_baseline(arm, target_s, gpu_dec):
    """The reference's own predict + schedule_d_dvfs (oracle/_ref, compiled
    from the reference sources) on 1 host thread over a bounded sample of the
    same workload (the first apps of rank 0's shard)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O

    g, sc = arm.g, arm.sc
    budgets = arm.budgets
    if O.ref_available():
        probe = 2
        secs, _ = O.ref_bench_grid(sc.energy, sc.time, g, budgets, probe, 1)
        n = int(max(2, min(arm.A, target_s / max(secs / probe, 1e-6))))
        secs, dec = O.ref_bench_grid(sc.energy, sc.time, g, budgets, n, 1)
        kind = "reference"
    else:
        t0 = time.perf_counter()
        O.oracle_grid(sc.energy, sc.time, g, budgets, app_slice=(0, 2))
        per = (time.perf_counter() - t0) / 2
        n = int(max(2, min(arm.A, target_s / max(per, 1e-6))))
        t0 = time.perf_counter()
        dec, _, _ = O.oracle_grid(sc.energy, sc.time, g, budgets, app_slice=(0, n))
        secs = time.perf_counter() - t0
        kind = "port"
    match = bool(np.array_equal(dec.view(np.uint8), gpu_dec[:n].view(np.uint8)))
    return {"value": n * g.n_clocks / secs, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"first {n} apps x {g.n_clocks} clocks ({n * g.n_clocks} predictions) of the same workload "
                      f"and deadlines: materialised rows -> models::predict (E, T) -> "
                      f"schedule_d_dvfs(full_deadline); {secs:.1f} s; per-prediction rate extrapolates linearly to "
                      f"the full batch",
            "decisions_match_gpu": match}


def run_reference(args, rank, world):
    """The reference's CPU implementation (oracle/_ref: its own models::predict
    + schedule_d_dvfs compiled from its sources) on all host threads, on the
    same config, inputs and deadlines (a bounded sample of the batch per step,
    each thread on a contiguous app partition)."""
    if rank != 0:
        return None
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O

    cfg, per_rank, n_total = workload_config(args.config, world, args.apps)
    if not O.ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libgpudvfs_ref.so not built"}
    threads = os.cpu_count() or 1
    # sample size: probe the per-app cost on a few apps
    probe_n = min(threads, 64)
    sc, budgets = cpu_sample_grid(cfg, n_total, probe_n, args.w_clk)
    secs, _ = O.ref_bench_grid(sc.energy, sc.time, sc.grid, budgets, probe_n, threads)
    per_step_target = max(1.0, min(6.0, 150.0 / max(args.steps + args.warmup, 1)))
    n = int(max(threads, min(n_total, 1 << 16, per_step_target / max(secs / probe_n, 1e-9))))
    sc, budgets = cpu_sample_grid(cfg, n_total, n, args.w_clk)
    g = sc.grid
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
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (the same chunk-seeded inputs and deadlines)",
        "config": config_json(args.config, cfg, per_rank, n_total, world, g.n_clocks),
        "decisions_per_s": n / step_s,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"first {n} of the {n_total} apps x {g.n_clocks} clocks per step, {threads} "
                                   "threads on contiguous app partitions: materialised rows -> models::predict "
                                   "(E, T) -> schedule_d_dvfs(full_deadline); rate extrapolates linearly"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


FACADE = ROOT / "integration" / "_build" / "facade_test"


def run_c1(args, impl):
    """BASELINE configs[0], the paper-scale production path: the P100 catalog
    (12 suite apps x 62 clocks, profiled at every other clock), fit_gbt 100 x
    depth 10 energy + time, k-means clusters, then a cold make_model_predictor
    + schedule_d_dvfs(full_deadline) over the job batch -- through the C++
    drop-in (gpu_api.hpp) and through the reference's own functions, in one
    process on the same inputs (integration/facade_test --bench).  Decisions
    must be identical.  Host-side work (correlation, encoding, EDF) dominates
    at this size; the GPU evaluates the 62 x 100-tree candidates."""
    jobs = args.apps or 100
    reps = max(1, args.steps)
    if not FACADE.exists():
        return {"impl": impl, "unavailable": "integration/_build/facade_test not built (needs the reference headers)"}
    r = subprocess.run([str(FACADE), "--bench", str(reps), "100", "10", str(jobs)], capture_output=True, text=True,
                       timeout=1800)
    if r.returncode != 0:
        raise RuntimeError(f"facade bench failed: {r.stdout[-500:]} {r.stderr[-500:]}")
    d = json.loads(r.stdout.strip().splitlines()[-1])
    preds = d["jobs"] * d["clocks"]
    ms = d["reference_ms_median"] if impl == "reference" else d["dropin_ms_median"]
    value = preds / (ms * 1e-3)
    cfg = {"workload": f"BASELINE configs[0] (c1): paper-scale production path, P100 catalog "
                       f"({d['catalog_records']} profiled records, {d['clocks']} clocks), fit_gbt {d['trees']} trees "
                       f"depth {d['depth']} E + T, {d['jobs']}-job batch, cold predictor + schedule_d_dvfs "
                       f"(full_deadline)", "jobs": d["jobs"], "clocks": d["clocks"], "parallelism": "dp1",
           "api": "C++ drop-in gpu::make_model_predictor + gpu::schedule_d_dvfs" if impl != "reference" else
                  "reference sched::make_model_predictor + sched::schedule_d_dvfs"}
    res = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": reps, "warmup": 1,
           "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (the reference's own synthetic P100 GPU and suite; queries seeded)", "config": cfg,
           "decisions_per_s": d["jobs"] / (ms * 1e-3),
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                   "note": "the C++ API call itself is the end-to-end path (host tables in, decisions out)"},
           "decisions_identical_to_reference": d["decisions_identical"], "scheduled": d["scheduled"],
           "facade": d}
    if impl == "reference":
        res["impl"] = "reference"
        res["cpu_baseline"] = {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                               "sample": f"the whole {d['jobs']}-job batch"}
        res["e2e"]["h2d_bytes_per_step"] = res["e2e"]["d2h_bytes_per_step"] = 0
    else:
        res["cpu_baseline"] = {"value": preds / (d["reference_ms_median"] * 1e-3), "unit": UNIT, "cores": 1,
                               "kind": "reference", "sample": f"the whole {d['jobs']}-job batch, same process"}
    return res


def main():
    args = parse_args()
    if args.config == "c1":
        print(json.dumps(run_c1(args, args.impl)), flush=True)
        return
    if args.gpus > 1 and "RANK" not in os.environ:
        # One process per GPU: re-execute under torch.distributed.run.
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, world, local_rank)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
