"""Small workloads through every kernel of the token-layout path, for compute-sanitizer.

    compute-sanitizer --tool memcheck|synccheck|racecheck python tools/sanitize_path.py

Runs SparseAttention (tokens and tiled modes) on toy shapes with ragged grids, mixed
per-head tile shapes and both token layouts, the host-buffer pipeline, and the warp /
CTA top-k kernels; prints one line per case.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import synth, veda  # noqa: E402


def main():
    veda.load()
    dev = torch.device("cuda")
    cases = [("tiny", (4, 8, 8), [(4, 4, 4)], 64, 1, 0.5),
             ("ragged_b128", (5, 9, 14), [(4, 4, 8)], 128, 2, 0.5),
             ("mixed", (9, 10, 13), [(4, 4, 8), (8, 4, 4), (4, 8, 4), (8, 8, 2)], 128, 4, 0.8),
             ("b64_d128", (3, 5, 6), [(4, 4, 4)], 128, 2, 0.5)]
    for name, lat, cfgs, d, Hh, sp in cases:
        cf = cfgs * Hh if len(cfgs) == 1 else cfgs
        pre = synth.Preset(name, lat, Hh, d, cf[0], sp)
        q, k, v = synth.qkv(pre, lat=lat, d=d)
        w = {n: t.to(dev) for n, t in synth.scorer_weights(pre, d=d, random_bias=True).items()}
        for mode in ("tokens", "tiled"):
            path = veda.SparseAttention(lat, cf, Hh, d, w, sparsity=sp, device=dev, mode=mode)
            o = path(q.to(dev), k.to(dev), v.to(dev))
            qn, kn, vn = (t.transpose(0, 1).contiguous().to(dev).transpose(0, 1) for t in (q, k, v))
            o2 = path(qn, kn, vn, out=torch.empty_like(qn))
            torch.cuda.synchronize()
            assert torch.equal(o, o2.contiguous())
        oh = path.run_host(q.contiguous().pin_memory(), k.contiguous().pin_memory(), v.contiguous().pin_memory(),
                           heads_per_chunk=1)
        torch.cuda.synchronize()
        assert torch.equal(oh.view(torch.int16), o.cpu().view(torch.int16))
        print(f"{name}: ok (k={path.k}, n_tiles={path.shape.n_tiles})", flush=True)
    # unit shares (veda_tile_pool_heads + veda_sparse_attn_fwd_tokens_units) with per-head
    # tile shapes, shares split inside heads
    from paper_2605_30325_b200 import shard
    cfgs = [(4, 4, 8), (8, 4, 4), (4, 8, 4)]
    pre = synth.Preset("units", (9, 10, 13), 3, 128, cfgs[0], 0.8)
    q, k, v = (t.to(dev) for t in synth.qkv(pre, lat=(9, 10, 13), d=128))
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre, d=128, random_bias=True).items()}
    full = veda.SparseAttention((9, 10, 13), cfgs, 3, 128, w, sparsity=0.8, device=dev)
    want = full(q, k, v)
    NT = full.shape.n_tiles
    out = torch.zeros_like(q)
    for r in range(3):
        u = shard.unit_range(3, NT, r, 3)
        veda.SparseAttention((9, 10, 13), cfgs, 3, 128, w, sparsity=0.8, device=dev, units=(u.start, u.stop))(
            q, k, v, out=out)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), want.view(torch.int16))
    print("unit shares: ok", flush=True)
    # scorer at a size where the GELU split's blocks loop over several row groups (R = 2 x 1000
    # rows, 500 row groups > the resident grid)
    pre = synth.Preset("scorer", (8, 16, 16), 2, 128, (4, 4, 8), 0.5)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre, d=128, random_bias=True).items()}
    NT = 1000
    g = torch.Generator().manual_seed(5)
    zq, zk = (torch.randn(2, NT, 3 * 128, generator=g).to(dev) for _ in range(2))
    cnt = torch.full((2, NT), 128, dtype=torch.int32, device=dev)
    s1 = veda.tile_score_pooled(zq, zk, cnt, veda.make_scorer(w))
    torch.cuda.synchronize()
    assert torch.isfinite(s1).all()
    print(f"scorer NT={NT}: ok", flush=True)
    for NT, kk in ((300, 17), (2100, 50)):  # warp and CTA top-k kernels
        s = torch.randn(2, NT, NT, device=dev)
        veda.select_topk(s, kk)
        torch.cuda.synchronize()
        print(f"topk NT={NT}: ok", flush=True)


if __name__ == "__main__":
    main()
