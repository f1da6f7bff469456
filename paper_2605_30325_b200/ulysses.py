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


def chunk_range(hr: range, c: int, C: int) -> range:
    """Chunk c of C of a head range (sizes differ by at most one)."""
    n = len(hr)
    return range(hr.start + (c * n) // C, hr.start + ((c + 1) * n) // C)


def seq_to_head_async(x_local: torch.Tensor, lat, heads_of, group=None):
    """Start all-to-all #1 for the heads heads_of[j] of every rank j: returns (recv, work),
    recv = this rank's heads [N, len(heads_of[rank]), d] once work.wait() returns (for NCCL:
    once the current stream waits on it).  Rows arrive ordered by source rank = by token."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    Nr, Hh, d = x_local.shape
    counts = token_counts(lat, world)
    assert Nr == counts[rank], (Nr, counts)
    send = torch.cat([_payload(x_local[:, hj.start:hj.stop, :]).reshape(-1) for hj in heads_of])
    dp = d * x_local.element_size() // send.element_size()  # payload elements per row
    my = heads_of[rank]
    recv = torch.empty(sum(counts) * len(my) * dp, dtype=send.dtype, device=send.device)
    work = dist.all_to_all_single(recv, send, output_split_sizes=[c * len(my) * dp for c in counts],
                                  input_split_sizes=[Nr * len(hj) * dp for hj in heads_of], group=group,
                                  async_op=True)
    return _restore(recv.view(sum(counts), len(my), dp), x_local), work


def head_to_seq_async(o_heads: torch.Tensor, lat, heads_of, group=None):
    """Start all-to-all #2 of this rank's heads heads_of[rank] ([N, h, d]) back to the sequence
    shards: returns (place, work); after work.wait(), place(out) writes the received rows into
    out [N_r, Hh, d] (columns heads_of[j] of every source j)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    N, Hr, d = o_heads.shape
    counts = token_counts(lat, world)
    assert Hr == len(heads_of[rank])
    starts = [sum(counts[:i]) for i in range(world)]
    send = torch.cat([_payload(o_heads[starts[i]:starts[i] + counts[i]]).reshape(-1) for i in range(world)])
    dp = d * o_heads.element_size() // send.element_size()
    Nr = counts[rank]
    recv = torch.empty(Nr * sum(len(hj) for hj in heads_of) * dp, dtype=send.dtype, device=send.device)
    work = dist.all_to_all_single(recv, send, output_split_sizes=[Nr * len(hj) * dp for hj in heads_of],
                                  input_split_sizes=[c * Hr * dp for c in counts], group=group, async_op=True)

    def place(out):
        ov = _payload(out) if out.element_size() == 2 else out
        ov = ov.view(Nr, -1, dp)
        off = 0
        for hj in heads_of:
            n = Nr * len(hj) * dp
            ov[:, hj.start:hj.stop, :] = recv[off:off + n].view(Nr, len(hj), dp)
            off += n

    place.recv = recv  # callers that place on another stream record it there (record_stream)
    return place, work


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
    (head_range(Hh, rank, G)).  Every rank's head range is computed on the WHOLE call's
    padded grid (SparseAttention(head_range=...)), so the output equals the single-GPU call
    bit for bit, head-aware tiling included.

    chunks = C > 1 overlaps the exchange with the path: each rank's
    heads are cut into C chunks; all 3C input all-to-alls (Q, K, V of each chunk) are started
    at once, the path of chunk c runs as soon as its own three have landed -- while those of
    chunks c+1.. are still in flight on the communicator's stream -- and the output
    all-to-all of chunk c starts as soon as its path is done, overlapping chunk c+1's path."""

    def __init__(self, lat, cfgs, Hh, d, scorer_weights, sparsity=None, k=None, group=None, device="cuda",
                 chunks: int = 1):
        from . import veda

        self.lat, self.Hh, self.group = tuple(lat), Hh, group
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        self.world, self.rank = world, rank
        self.heads = head_range(Hh, rank, world)
        self.chunks = max(1, int(chunks))
        cf = list(cfgs)
        if len(cf) == 1:
            cf = cf * Hh
        # the padded grid, N_T and k are the WHOLE call's (all Hh configs), so every rank's
        # heads are computed exactly as in the single-GPU call even with head-aware tiling
        self.paths = []
        for c in range(self.chunks):
            hc = chunk_range(self.heads, c, self.chunks)
            a, b = hc.start - self.heads.start, hc.stop - self.heads.start
            w = {n: t[a:b] for n, t in scorer_weights.items()}
            self.paths.append(veda.SparseAttention(lat, cf, Hh, d, w, sparsity=sparsity, k=k, device=device,
                                                   head_range=hc))
        self.path = self.paths[0]

    def __call__(self, q, k, v, trace=None):
        """``trace`` (optional list): (label, torch.cuda.Event) pairs recorded on the current
        stream -- start, each chunk's inputs usable / path done, the end -- for overlap
        timelines (tools/ulysses_overlap.py).

        Streams: the send buffers of every chunk are packed and their all-to-alls issued on a
        side stream ``xs`` (in chunk order, so chunk 0 lands first); the caller's stream runs
        chunk c's path as soon as chunk c's three exchanges are done; chunk c's output
        exchange (pack + all-to-all) is issued on a second side stream ``xo`` once its path
        is done; the received rows are placed into ``out`` on the caller's stream at the end."""
        C, G = self.chunks, self.world
        cs = torch.cuda.current_stream(q.device)
        if not hasattr(self, "_xs"):
            self._xs, self._xo = torch.cuda.Stream(device=q.device), torch.cuda.Stream(device=q.device)
        xs, xo = self._xs, self._xo

        def mark(label):
            if trace is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(cs)
                trace.append((label, e))

        mark("start")
        heads_of = [[chunk_range(head_range(self.Hh, j, G), c, C) for j in range(G)] for c in range(C)]
        xs.wait_stream(cs)  # q, k, v are ready on the caller's stream
        with torch.cuda.stream(xs):
            ins = [[seq_to_head_async(t, self.lat, heads_of[c], self.group) for t in (q, k, v)] for c in range(C)]
        for c in range(C):
            for r, _ in ins[c]:
                r.record_stream(cs)  # allocated on xs, read by the path on cs
        mark("inputs issued")
        outs = []
        for c in range(C):
            for _, work in ins[c]:
                work.wait()  # the caller's stream waits for chunk c's exchanges only
            mark(f"chunk {c} inputs in")
            qh, kh, vh = (r for r, _ in ins[c])  # [N, h_c, d]
            o = torch.empty_like(qh)
            if qh.shape[1]:
                # the path reads/writes [h_c, N, d] views of the [N, h_c, d] buffers (strided, no copy)
                self.paths[c](qh.transpose(0, 1), kh.transpose(0, 1), vh.transpose(0, 1), out=o.transpose(0, 1))
            mark(f"chunk {c} path done")
            xo.wait_stream(cs)
            o.record_stream(xo)
            with torch.cuda.stream(xo):
                place, work = head_to_seq_async(o, self.lat, heads_of[c], self.group)
            place.recv.record_stream(cs)  # allocated on xo, read by place() on cs
            outs.append((place, work))
        out = torch.empty_like(q)
        for place, work in outs:
            work.wait()
            place(out)
        mark("end")
        return out
