"""Data-parallel sharding for multi-GPU decode.

Images are independent, so each rank decodes its own shard of the
dataset with no collective on the decode path. torch.distributed is used only for
plumbing outside the timed region: a barrier and the max-over-ranks of the
elapsed device time (one process per GPU, NCCL on B200; gloo in CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(num_items: int, rank: int, world: int) -> range:
    """Contiguous, balanced shard of [0, num_items) for `rank` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(num_items, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def shard_by_bytes(sizes, world: int) -> list[list[int]]:
    """Greedy longest-first assignment of items (e.g. compressed file sizes) to ranks,
    balancing total bytes (variable-size ImageNet-shaped batches)."""
    order = sorted(range(len(sizes)), key=lambda i: -sizes[i])
    load = [0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda q: (load[q], q))
        out[r].append(i)
        load[r] += sizes[i]
    return [sorted(s) for s in out]


def _device_for_backend():
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def max_over_ranks(value: float) -> float:
    """Max of a per-rank scalar (e.g. elapsed ms) over all ranks; identity without a process group."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for_backend())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float) -> float:
    """Sum of a per-rank scalar (e.g. algorithmic bytes) over all ranks; identity without a process group."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for_backend())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def all_ranks_true(flag: bool) -> bool:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return bool(flag)
    t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=_device_for_backend())
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def aggregate_throughput(units_per_rank: int, world: int, steps: int, max_ms: float) -> float:
    """Whole-job throughput: units all ranks processed / max-over-ranks elapsed seconds."""
    return units_per_rank * world * steps / (max_ms / 1e3)
