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


@pytest.mark.parametrize("preset,head_aware", [("wan1.3b", False), ("wan1.3b", True)])
def test_ulysses_nccl_world1_equals_direct(preset, head_aware):
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
        up = ulysses.UlyssesSparseAttention(pre.lat, cfgs, pre.heads, pre.d, w, sparsity=pre.sparsity, device=dev)
        o_u = up(q, k, v)
        path = veda.SparseAttention(pre.lat, cfgs, pre.heads, pre.d, w, sparsity=pre.sparsity, device=dev)
        o_d = path(q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1))  # [Hh, N, d]
        torch.cuda.synchronize()
        assert torch.equal(o_u.view(torch.int16), o_d.transpose(0, 1).contiguous().view(torch.int16))
        assert torch.equal(up.path.idx, path.idx)
    finally:
        dist.destroy_process_group()
