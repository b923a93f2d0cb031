"""Query-row sharding across the GPUs of one box.

Apps are independent under ``DeadlineBudget::full_deadline`` (each decision
depends only on the app's row, the models and its deadline,
scheduler.cpp:203-205), so rank g of G evaluates the contiguous app range
``[g*A/G, (g+1)*A/G)`` with its own replica of the packed models.  The one
collective is the gather of the 24-byte per-app decision records: on GPUs
the library's own NCCL gather to rank 0 (gd_gather_decisions / gd.Comm,
what bench.py uses); here its torch.distributed mirror for CPU tests (gloo),
with the same rank-order layout.
"""
from __future__ import annotations

from typing import Tuple

DECISION_BYTES = 24


def shard_range(n_apps: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) app range of `rank`; sizes differ by at most one."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n_apps * rank // world, n_apps * (rank + 1) // world


def gather_decisions(local, n_apps: int, world: int, group=None):
    """All-gather each rank's decision bytes (uint8 tensor of
    DECISION_BYTES * local_apps) and return the full batch in app order.

    Shards may differ by one app; every rank pads to the largest shard so
    the collective moves equal-sized buffers, then the padding is dropped.
    """
    import torch
    import torch.distributed as dist

    sizes = [shard_range(n_apps, r, world) for r in range(world)]
    max_apps = max(hi - lo for lo, hi in sizes)
    buf = torch.zeros(max_apps * DECISION_BYTES, dtype=torch.uint8, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[: (hi - lo) * DECISION_BYTES] for p, (lo, hi) in zip(parts, sizes)])


def shard_counts(n_apps: int, world: int):
    """Apps per rank, in rank order (the counts gd_gather_decisions takes)."""
    return [hi - lo for lo, hi in (shard_range(n_apps, r, world) for r in range(world))]


def gather_decisions_to_root(local, n_apps: int, world: int, root: int = 0, group=None):
    """gd_gather_decisions' semantics over torch.distributed: every rank's
    decision bytes land on `root` in rank order (None on the other ranks).
    Shards are padded to the largest so the collective moves equal sizes."""
    import torch
    import torch.distributed as dist

    counts = shard_counts(n_apps, world)
    max_apps = max(counts)
    buf = torch.zeros(max_apps * DECISION_BYTES, dtype=torch.uint8, device=local.device)
    buf[: local.numel()] = local
    rank = dist.get_rank(group)
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == root else None
    dist.gather(buf, parts, dst=root, group=group)
    if rank != root:
        return None
    return torch.cat([p[: c * DECISION_BYTES] for p, c in zip(parts, counts)])
