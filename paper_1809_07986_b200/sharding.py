"""Multi-GPU data parallelism over independent sequences.

Sequences are recursive in time but mutually independent, so the batch is
split into contiguous shards, one per rank (one process per GPU). There is no
collective on the data path; the only exchange is a final gather of a few
per-rank statistics (frames, cells, device time) — NCCL over NVLink on the GPU
box, gloo in the CPU tests. Timing is the max over ranks.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass


def shard(n_items: int, world: int, rank: int) -> range:
    """Contiguous shard of ``n_items`` for ``rank`` of ``world``; the first
    ``n_items % world`` ranks take one extra item."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard: bad world/rank")
    base, rem = divmod(n_items, world)
    start = rank * base + min(rank, rem)
    return range(start, start + base + (1 if rank < rem else 0))


@dataclass
class RankStats:
    rank: int
    sequences: int
    frames: int
    cells: float
    device_ms: float


def gather_stats(stats: RankStats, device=None) -> list[RankStats] | None:
    """All ranks' stats on every rank (all_gather of a small float tensor).
    Returns ``[stats]`` when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return [stats]
    world = dist.get_world_size()
    t = torch.tensor([float(v) for v in asdict(stats).values()], dtype=torch.float64,
                     device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    rows = [o.cpu().tolist() for o in out]
    return [RankStats(int(r[0]), int(r[1]), int(r[2]), r[3], r[4]) for r in rows]


def job_throughput(all_stats: list[RankStats]) -> dict:
    """Whole-job numbers: frames and cells of all ranks over the max device time."""
    t = max(s.device_ms for s in all_stats)
    frames = sum(s.frames for s in all_stats)
    cells = sum(s.cells for s in all_stats)
    return {"frames_per_s": frames / (t * 1e-3) if t > 0 else 0.0,
            "gcells_per_s": cells / (t * 1e-3) / 1e9 if t > 0 else 0.0,
            "max_device_ms": t, "frames": frames, "cells": cells}
