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


def unit_range(Hh: int, n_tiles: int, rank: int, world: int) -> range:
    """Rank r's contiguous share of the flattened (head, query tile) units u = h * n_tiles + i
    (SURVEY.md §8(e)'s finer partition): sizes differ by at most one unit, so head counts
    that do not divide the GPU count stay balanced (Wan-1.3B: 12 heads on 8 GPUs)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    n = Hh * n_tiles
    return range((rank * n) // world, ((rank + 1) * n) // world)


def heads_of_units(units: range, n_tiles: int) -> range:
    """Heads a unit share touches (their scores and lists are needed for its query tiles)."""
    if len(units) == 0:
        return range(0)
    return range(units.start // n_tiles, (units.stop - 1) // n_tiles + 1)


def max_over_ranks(value: float, group=None) -> float:
    """Device timings are reported as the max over ranks (all_reduce MAX)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
