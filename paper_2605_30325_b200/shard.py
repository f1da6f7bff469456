"""Head sharding across ranks.

Heads are independent in Veda (distinct phi per head; per-head loop in
Alg. 2), so rank r of G owns the contiguous global heads
[floor(r*Hh/G), floor((r+1)*Hh/G)) and the path needs no data-path collective.
"""
from __future__ import annotations


def head_range(Hh: int, rank: int, world: int) -> range:
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return range((rank * Hh) // world, ((rank + 1) * Hh) // world)


def max_over_ranks(value: float, group=None) -> float:
    """Device timings are reported as the max over ranks (all_reduce MAX)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
