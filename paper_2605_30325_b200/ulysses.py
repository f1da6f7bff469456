"""Ulysses-style sequence parallelism around the head-sharded path.

A DiT that shards its activations by sequence holds, on rank r of G, the tokens of whole
latent frames [T_r0, T_r1) for ALL heads: x_local [N_r, Hh, d].  Veda's path works per
head, so one all-to-all (NCCL over NVLink; gloo on CPU) turns the
sequence shard into a head shard [N, Hh_r, d] (rank r keeps heads head_range(Hh, r, G)),
the local path runs on full sequences, and a second all-to-all returns the output to the
sequence shard.  The exchange is the only collective; the path itself has none
("SP=8" names the setting but not its mechanism).

The exchange functions are device-agnostic and carry raw 16-bit payloads, so the same
code is exercised by the world-size-2 gloo test on CPU and by NCCL on B200s.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .shard import head_range


def frame_range(T: int, rank: int, world: int) -> range:
    """Latent frames owned by `rank` (whole frames; sequence shards follow frame bounds)."""
    return range((rank * T) // world, ((rank + 1) * T) // world)


def token_counts(lat, world: int):
    T, H, W = lat
    return [len(frame_range(T, r, world)) * H * W for r in range(world)]


def _payload(x: torch.Tensor) -> torch.Tensor:
    """Raw view for the exchange: 16-bit rows travel as int32 pairs (gloo has no 16-bit
    types; NCCL moves the same bytes)."""
    if x.element_size() == 2:
        return x.contiguous().view(torch.int32)
    return x.contiguous()


def _restore(p: torch.Tensor, like: torch.Tensor) -> torch.Tensor:
    return p.view(like.dtype) if like.element_size() == 2 else p


def seq_to_head(x_local: torch.Tensor, lat, group=None) -> torch.Tensor:
    """[N_r, Hh, d] sequence shard -> [N, Hh_r, d] head shard (all-to-all #1)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    Nr, Hh, d = x_local.shape
    counts = token_counts(lat, world)
    assert Nr == counts[rank], (Nr, counts)
    heads = [head_range(Hh, j, world) for j in range(world)]
    send = torch.cat([_payload(x_local[:, hj.start:hj.stop, :]).reshape(-1) for hj in heads])
    dp = d * x_local.element_size() // send.element_size()  # payload elements per row
    my = heads[rank]
    recv = torch.empty(sum(counts) * len(my) * dp, dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send, output_split_sizes=[c * len(my) * dp for c in counts],
                           input_split_sizes=[Nr * len(hj) * dp for hj in heads], group=group)
    return _restore(recv.view(sum(counts), len(my), dp), x_local)


def head_to_seq(o_heads: torch.Tensor, lat, Hh: int, group=None) -> torch.Tensor:
    """[N, Hh_r, d] head shard -> [N_r, Hh, d] sequence shard (all-to-all #2)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    N, Hr, d = o_heads.shape
    counts = token_counts(lat, world)
    heads = [head_range(Hh, j, world) for j in range(world)]
    assert Hr == len(heads[rank])
    starts = [sum(counts[:i]) for i in range(world)]
    send = torch.cat([_payload(o_heads[starts[i]:starts[i] + counts[i]]).reshape(-1) for i in range(world)])
    dp = d * o_heads.element_size() // send.element_size()
    Nr = counts[rank]
    recv = torch.empty(Nr * Hh * dp, dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send, output_split_sizes=[Nr * len(hj) * dp for hj in heads],
                           input_split_sizes=[c * Hr * dp for c in counts], group=group)
    out = torch.empty((Nr, Hh, dp), dtype=send.dtype, device=send.device)
    off = 0
    for hj in heads:
        n = Nr * len(hj) * dp
        out[:, hj.start:hj.stop, :] = recv[off:off + n].view(Nr, len(hj), dp)
        off += n
    return _restore(out, o_heads)


class UlyssesSparseAttention:
    """Sequence-sharded front end of veda.SparseAttention (one instance per rank).

    __call__(q, k, v) takes [N_r, Hh, d] bf16 CUDA tensors (this rank's frames, all heads)
    and returns o [N_r, Hh, d]; scorer_weights hold this rank's heads
    (head_range(Hh, rank, G))."""

    def __init__(self, lat, cfgs, Hh, d, scorer_weights, sparsity=None, k=None, group=None, device="cuda"):
        from . import veda

        self.lat, self.Hh, self.group = tuple(lat), Hh, group
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        self.heads = head_range(Hh, rank, world)
        cf = list(cfgs)
        if len(cf) > 1:
            cf = cf[self.heads.start:self.heads.stop]
        self.path = veda.SparseAttention(lat, cf, len(self.heads), d, scorer_weights, sparsity=sparsity, k=k,
                                         device=device)

    def __call__(self, q, k, v):
        qh, kh, vh = (seq_to_head(t, self.lat, self.group) for t in (q, k, v))  # [N, Hh_r, d]
        o = torch.empty_like(qh)
        # the path reads/writes [Hh_r, N, d] views of the [N, Hh_r, d] buffers (strided, no copy)
        self.path(qh.transpose(0, 1), kh.transpose(0, 1), vh.transpose(0, 1), out=o.transpose(0, 1))
        return head_to_seq(o, self.lat, self.Hh, self.group)
