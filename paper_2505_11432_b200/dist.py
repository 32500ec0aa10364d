"""Host-side multi-rank plumbing shared by the layer, the attention
projections and bench.py (one process per GPU, torch.distributed for
bootstrap only; the data path runs over NVLink inside the kernels).

Partitioning follows the reference exactly:
  token t lives on rank t * n // T      (routing.cpp:81)
  expert j lives on rank j // (E / n)   (routing.cpp:44-47, routing.hpp:34-35)
"""
from __future__ import annotations

import torch


def token_owner(t: int, T: int, n: int) -> int:
    return t * n // max(T, 1)


def expert_owner(j: int, E: int, n: int) -> int:
    if E % n:
        raise ValueError("num_experts must be divisible by n")
    return j // (E // n)


def local_experts(rank: int, E: int, n: int) -> range:
    el = E // n
    return range(rank * el, (rank + 1) * el)


def exchange_blobs(blob: bytes, world: int, group=None) -> bytes:
    """All-gather one opaque blob per rank (CUDA IPC handles); returns the
    concatenation in rank order. Every blob must have the same length."""
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, blob, group=group)
    if len({len(b) for b in out}) != 1:
        raise RuntimeError("IPC handle blobs differ in size across ranks")
    return b"".join(out)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank timing (multi-GPU numbers are max over ranks)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
