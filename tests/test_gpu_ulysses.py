"""Ulysses front end on the GPU: NCCL all-to-alls (world size 1 on the single-GPU box) around
the token-layout path, which then reads the [N, Hh, d] exchange buffers through strided
[Hh, N, d] views (token-major 5-D TMA boxes).  Must equal the direct path bit for bit.
The multi-rank exchange logic itself is covered by tests/test_dist_gloo.py (world size 2)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("preset,head_aware,chunks", [("wan1.3b", False, 1), ("wan1.3b", True, 1),
                                                     ("wan1.3b", True, 3), ("wan1.3b", True, 16)])
def test_ulysses_nccl_world1_equals_direct(preset, head_aware, chunks):
    from paper_2605_30325_b200 import build, synth, ulysses, veda

    build.build()
    veda.load()
    pre = synth.PRESETS[preset]
    cfgs = [synth.HEAD_AWARE_CFGS[h % 4] for h in range(pre.heads)] if head_aware else [pre.cfg]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        w = {n: t.to(dev) for n, t in synth.scorer_weights(pre).items()}
        q, k, v = synth.qkv(pre, device=dev, layout="nhd")  # [N, Hh, d] sequence layout
        up = ulysses.UlyssesSparseAttention(pre.lat, cfgs, pre.heads, pre.d, w, sparsity=pre.sparsity, device=dev,
                                            chunks=chunks)
        o_u = up(q, k, v)
        path = veda.SparseAttention(pre.lat, cfgs, pre.heads, pre.d, w, sparsity=pre.sparsity, device=dev)
        o_d = path(q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1))  # [Hh, N, d]
        torch.cuda.synchronize()
        assert torch.equal(o_u.view(torch.int16), o_d.transpose(0, 1).contiguous().view(torch.int16))
        if chunks == 1:
            assert torch.equal(up.path.idx, path.idx)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G", [2, 5, 8, 16])
def test_head_range_shards_equal_single_gpu_call(G):
    """What each Ulysses rank computes (SparseAttention(head_range=...) on its [N, Hh/G, d]
    head shard, the exchange's output) assembles to the single-GPU call bit for bit with
    head-aware per-head tile shapes -- the padded grid, N_T and k are the whole call's, not
    those of the rank's own heads.  G = 16 > 12 heads leaves ranks without heads."""
    from paper_2605_30325_b200 import build, shard, synth, veda

    build.build()
    veda.load()
    pre = synth.PRESETS["wan1.3b"]
    cfgs = [synth.HEAD_AWARE_CFGS[h % 4] for h in range(pre.heads)]
    dev = torch.device("cuda", 0)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre).items()}
    q, k, v = synth.qkv(pre, device=dev, layout="nhd")  # [N, Hh, d]
    full = veda.SparseAttention(pre.lat, cfgs, pre.heads, pre.d, w, sparsity=pre.sparsity, device=dev)
    want = full(q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1))
    got = torch.full_like(q, 3.0)
    for r in range(G):
        hr = shard.head_range(pre.heads, r, G)
        wr = {n: t[hr.start:hr.stop] for n, t in w.items()}
        qs, ks, vs = (t[:, hr.start:hr.stop].contiguous() for t in (q, k, v))  # the exchange's [N, Hh_r, d]
        pr = veda.SparseAttention(pre.lat, cfgs, pre.heads, pre.d, wr, sparsity=pre.sparsity, device=dev,
                                  head_range=hr)
        assert pr.k == full.k and pr.shape.n_tiles == full.shape.n_tiles
        o = torch.empty_like(qs)
        pr(qs.transpose(0, 1), ks.transpose(0, 1), vs.transpose(0, 1), out=o.transpose(0, 1))
        got[:, hr.start:hr.stop] = o
        if len(hr):
            assert torch.equal(pr.idx, full.idx[hr.start:hr.stop])
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.int16), want.transpose(0, 1).contiguous().view(torch.int16))
