"""Multi-process (world size 2, gloo, CPU) coverage of the N>1 path: head sharding
(paper_2605_30325_b200/shard.py) and the max-over-ranks timing reduction.  The fp64
oracle stands in for the CUDA kernels; per-head results of the sharded run must be
bit-identical to the single-process run (heads are independent)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

LAT = (5, 7, 9)
CFGS = [(2, 4, 2), (4, 2, 2), (1, 4, 4)]
D, KK = 8, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _path_for_heads(heads):
    """The whole path (oracle backend) for the given global heads."""
    import oracle
    from paper_2605_30325_b200 import synth

    oracle.build()
    pre = synth.Preset("dist", LAT, len(CFGS), D, CFGS[0], 0.5)
    q, k, v = synth.qkv(pre, heads=heads, lat=LAT, d=D, alpha=2.0)
    w = synth.scorer_weights(pre, heads=heads, d=D, random_bias=True)
    u = lambda t: t.contiguous().view(torch.int16).numpy().view(np.uint16)
    cf = [CFGS[h] for h in heads]
    # the padded grid must be the one of the WHOLE call (all heads), so pass every config
    # and keep the local heads' rows
    allq = np.zeros((len(CFGS),) + tuple(q.shape[1:]), np.uint16)
    allk, allv = allq.copy(), allq.copy()
    for li, h in enumerate(heads):
        allq[h], allk[h], allv[h] = u(q[li]), u(k[li]), u(v[li])
    oq, cnt, mask = oracle.tile_permute(allq, LAT, CFGS)
    ok_, _, _ = oracle.tile_permute(allk, LAT, CFGS)
    ov, _, _ = oracle.tile_permute(allv, LAT, CFGS)
    sel = list(heads)
    oq, ok_, ov, cnt, mask = oq[sel], ok_[sel], ov[sel], cnt[sel], mask[sel]
    wn = {n: t.numpy() for n, t in w.items()}
    eq = oracle.mlp(oracle.trippool(oq, mask), wn["w1q"], wn["b1q"], wn["w2q"], wn["b2q"])
    ek = oracle.mlp(oracle.trippool(ok_, mask), wn["w1k"], wn["b1k"], wn["w2k"], wn["b2k"])
    s = oracle.scores(eq, ek, cnt)
    idx = oracle.topk(s.astype(np.float32).astype(np.float64), KK)
    o = oracle.sparse_attn(oq, ok_, ov, idx, mask, nthreads=1)
    return {"idx": idx, "o": o, "s": s}


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_30325_b200 import shard

    heads = shard.head_range(len(CFGS), rank, world)
    res = _path_for_heads(list(heads))
    gathered = [None] * world
    dist.all_gather_object(gathered, (list(heads), res))
    t = shard.max_over_ranks(float(rank + 1) * 1.5)
    if rank == 0:
        np.save(os.path.join(out_dir, "max.npy"), np.array([t]))
        for hs, r in gathered:
            for li, h in enumerate(hs):
                np.save(os.path.join(out_dir, f"idx{h}.npy"), r["idx"][li])
                np.save(os.path.join(out_dir, f"o{h}.npy"), r["o"][li])
    dist.barrier()
    dist.destroy_process_group()


def test_head_range_partition():
    from paper_2605_30325_b200 import shard

    for Hh in (1, 3, 12, 24, 40):
        for G in (1, 2, 4, 8):
            parts = [list(shard.head_range(Hh, r, G)) for r in range(G)]
            assert sum(parts, []) == list(range(Hh))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
    assert [len(shard.head_range(24, r, 8)) for r in range(8)] == [3] * 8


def test_unit_range_partition():
    """The finer (head x query tile) share: every unit exactly once, sizes within one, and
    the heads a share touches are exactly those of its units."""
    from paper_2605_30325_b200 import shard

    for Hh, NT in ((12, 336), (24, 1920), (3, 7), (1, 5), (40, 720)):
        for G in (1, 2, 3, 4, 8):
            parts = [shard.unit_range(Hh, NT, r, G) for r in range(G)]
            assert sum((list(p) for p in parts), []) == list(range(Hh * NT))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
            for p in parts:
                assert list(shard.heads_of_units(p, NT)) == sorted({u // NT for u in p})
    # Wan-1.3B on 8 GPUs: head sharding leaves the busiest rank 2 of 12 heads, units 1.5
    assert max(len(shard.head_range(12, r, 8)) for r in range(8)) == 2
    assert max(len(shard.unit_range(12, 336, r, 8)) for r in range(8)) == 12 * 336 // 8


def _unit_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_30325_b200 import shard

    import oracle

    oracle.build()
    full = _path_for_heads(list(range(len(CFGS))))  # every rank may read the inputs of any head
    NT = full["o"].shape[1]
    units = shard.unit_range(len(CFGS), NT, rank, world)
    heads = shard.heads_of_units(units, NT)
    res = _path_for_heads(list(heads))  # scores / lists / attention of the touched heads only
    share = {}
    for u in units:
        h, i = divmod(u, NT)
        share[u] = (res["idx"][h - heads.start][i], res["o"][h - heads.start][i])
    gathered = [None] * world
    dist.all_gather_object(gathered, share)
    if rank == 0:
        merged = {}
        for g in gathered:
            assert not (set(g) & set(merged))  # disjoint shares
            merged.update(g)
        np.save(os.path.join(out_dir, "units.npy"), np.array(sorted(merged)))
        np.save(os.path.join(out_dir, "idx.npy"), np.stack([merged[u][0] for u in sorted(merged)]))
        np.save(os.path.join(out_dir, "o.npy"), np.stack([merged[u][1] for u in sorted(merged)]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_unit_shares_equal_single(tmp_path):
    """Unit (head x query tile) shares, assembled, equal the single-process call unit by unit
    (world size 2: the split falls inside a head, whose K side both ranks then compute)."""
    world, port = 2, _free_port()
    mp.spawn(_unit_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    single = _path_for_heads(list(range(len(CFGS))))
    Hh, NT = single["o"].shape[:2]
    assert np.array_equal(np.load(tmp_path / "units.npy"), np.arange(Hh * NT))
    assert np.array_equal(np.load(tmp_path / "idx.npy"), single["idx"].reshape(Hh * NT, -1))
    assert np.array_equal(np.load(tmp_path / "o.npy"), single["o"].reshape((Hh * NT,) + single["o"].shape[2:]),
                          equal_nan=True)


def test_gloo_world2_sharded_equals_single(tmp_path):
    world, port = 2, _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    single = _path_for_heads(list(range(len(CFGS))))
    assert float(np.load(tmp_path / "max.npy")[0]) == 3.0
    for h in range(len(CFGS)):
        assert np.array_equal(np.load(tmp_path / f"idx{h}.npy"), single["idx"][h])
        assert np.array_equal(np.load(tmp_path / f"o{h}.npy"), single["o"][h], equal_nan=True)


# --------------------------------------------------------------------------- Ulysses exchange

ULAT, UHH, UD = (5, 4, 6), 3, 8


def _global_tensor(seed):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn((ULAT[0] * ULAT[1] * ULAT[2], UHH, UD), generator=g) * 3).to(torch.bfloat16)


def _ulysses_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_30325_b200 import ulysses
    from paper_2605_30325_b200.shard import head_range

    x = _global_tensor(1)
    counts = ulysses.token_counts(ULAT, world)
    start = sum(counts[:rank])
    x_local = x[start:start + counts[rank]].contiguous()
    xh = ulysses.seq_to_head(x_local, ULAT)
    hr = head_range(UHH, rank, world)
    ok1 = torch.equal(xh.view(torch.int16), x[:, hr.start:hr.stop, :].contiguous().view(torch.int16))
    back = ulysses.head_to_seq(xh, ULAT, UHH)
    ok2 = torch.equal(back.view(torch.int16), x_local.view(torch.int16))
    # chunked exchange (the overlapped front end's): chunk c of every rank's heads
    ok3 = True
    for C in (2, 3, 4):
        heads_of = [[ulysses.chunk_range(head_range(UHH, j, world), c, C) for j in range(world)] for c in range(C)]
        got = [ulysses.seq_to_head_async(x_local, ULAT, heads_of[c]) for c in range(C)]
        out = torch.full_like(x_local, 7.0)
        for c in range(C):
            xc, w = got[c]
            w.wait()
            hc = heads_of[c][rank]
            ok3 &= torch.equal(xc.view(torch.int16), x[:, hc.start:hc.stop, :].contiguous().view(torch.int16))
            place, w2 = ulysses.head_to_seq_async(xc, ULAT, heads_of[c])
            w2.wait()
            place(out)
        ok3 &= torch.equal(out.view(torch.int16), x_local.view(torch.int16))
    # full path on the head shard with the oracle as the kernel backend, then back to sequence
    res = _path_on_heads(xh, hr)
    o_seq = ulysses.head_to_seq(res, ULAT, UHH)
    np.save(os.path.join(out_dir, f"o{rank}.npy"), o_seq.view(torch.int16).numpy())
    np.save(os.path.join(out_dir, f"ok{rank}.npy"), np.array([ok1, ok2, bool(ok3)]))
    dist.barrier()
    dist.destroy_process_group()


def _path_on_heads(x_heads, hr):
    """Oracle attention (dense over tiles, k = N_T) of [N, Hh_r, d] with q = k = v = x."""
    import oracle

    oracle.build()
    cfg = [(1, 2, 2)] * len(hr)
    xb = x_heads.transpose(0, 1).contiguous().view(torch.int16).numpy().view(np.uint16)
    xt, cnt, mask = oracle.tile_permute(xb, ULAT, cfg)
    NT = xt.shape[1]
    idx = np.broadcast_to(np.arange(NT, dtype=np.int32), (len(hr), NT, NT)).copy()
    o = oracle.sparse_attn(xt, xt, xt, idx, mask, nthreads=1)
    ob = oracle.tile_unpermute(oracle.f64_to_bf16_bits(o), ULAT, cfg)  # [Hh_r, N, d]
    return torch.from_numpy(ob.view(np.int16)).view(torch.bfloat16).transpose(0, 1).contiguous()


def test_ulysses_exchange_world2(tmp_path):
    world, port = 2, _free_port()
    mp.spawn(_ulysses_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    x = _global_tensor(1)
    full = _path_on_heads(x, range(UHH))  # single process, all heads
    counts = [len(range((r * ULAT[0]) // world, ((r + 1) * ULAT[0]) // world)) * ULAT[1] * ULAT[2] for r in range(world)]
    for r in range(world):
        assert np.load(tmp_path / f"ok{r}.npy").all()
        start = sum(counts[:r])
        want = full[start:start + counts[r]].view(torch.int16).numpy()
        assert np.array_equal(np.load(tmp_path / f"o{r}.npy"), want)
