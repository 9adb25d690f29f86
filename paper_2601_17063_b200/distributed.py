"""Multi-GPU sharding of the replay (north-star subsystem 4).

Every (trace, layer, policy, capacity) instance is independent (SURVEY.md
F3), so ranks replay disjoint shards with no data-path collective; the only
exchange is ONE all-reduce (NCCL over NVLink on the GPU box, gloo in the CPU
tests) of the int64 per-(policy, capacity) counters at the end.  Per-trace
float64 latencies are concatenated (all-gather of disjoint slots) rather
than summed, so every trace's SimReport stays bit-identical to a 1-GPU run.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block partition of n_items over world ranks: [begin, end)."""
    per = (n_items + world - 1) // world
    b = min(n_items, rank * per)
    return b, min(n_items, b + per)


def shard_layers(num_layers: int, rank: int, world: int) -> list[int]:
    """Round-robin layers (single-trace configs): layer l -> rank l % world."""
    return [l for l in range(num_layers) if l % world == rank]


def reduce_counters(counters: torch.Tensor) -> torch.Tensor:
    """Sum int64 counters [.., MCB_R_N] over ranks (the single collective).

    The status slot (index 7) is reduced with MAX so any failing cell
    surfaces; the others are summed.  Works for NCCL (CUDA tensors) and gloo
    (CPU tensors)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return counters
    status = counters[..., 7].clone()
    body = counters.clone()
    body[..., 7] = 0
    dist.all_reduce(body, op=dist.ReduceOp.SUM)
    dist.all_reduce(status, op=dist.ReduceOp.MAX)
    body[..., 7] = status
    return body


def gather_trace_rows(local: torch.Tensor, n_total: int, begin: int) -> torch.Tensor:
    """Place this rank's per-trace rows into a zeroed [n_total, ...] tensor and
    all-reduce: rows are disjoint, so the sum is a concatenation (exact)."""
    full = torch.zeros((n_total,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    full[begin:begin + local.shape[0]] = local
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(full, op=dist.ReduceOp.SUM)
    return full


def max_over_ranks(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
