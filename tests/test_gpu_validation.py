"""GPU: the boundary's index-list contract (exactly k distinct kept tiles per query tile,
ascending, reading R11) and input finiteness are checked on request and in
debug mode, and a bad list never makes the attention kernel read outside its head."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    from paper_2605_30325_b200 import build, veda

    build.build()
    veda.load()
    veda.check_device()
    return veda


@pytest.fixture(scope="module")
def case(V):
    from paper_2605_30325_b200 import synth

    pre = synth.Preset("val", (8, 16, 32), 2, 128, (4, 4, 8), 0.75)
    q, k, v = synth.qkv(pre)
    dev = torch.device("cuda")
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre).items()}
    path = V.SparseAttention(pre.lat, [pre.cfg], pre.heads, pre.d, w, sparsity=pre.sparsity, device=dev,
                             keep_scores=True)
    q, k, v = q.to(dev), k.to(dev), v.to(dev)
    o = path(q, k, v)
    torch.cuda.synchronize()
    return pre, path, q, k, v, o


def _bad_lists(idx, NT):
    out = {}
    a = idx.clone(); a[0, 3, 1] = NT; out["range_high"] = (a, "VEDA_ERR_INDEX")
    a = idx.clone(); a[1, 0, 0] = -1; out["range_negative"] = (a, "VEDA_ERR_INDEX")
    a = idx.clone(); a[0, 5, 2] = a[0, 5, 1]; out["duplicate"] = (a, "VEDA_ERR_INDEX")
    a = idx.clone(); a[1, 7] = torch.flip(a[1, 7], [0]); out["descending"] = (a, "VEDA_ERR_INDEX")
    return out


def test_validate_index_flags(V, case):
    pre, path, q, k, v, o = case
    NT = path.shape.n_tiles
    assert V.validate_index(path.idx, NT) == 0
    for name, (bad, _) in _bad_lists(path.idx, NT).items():
        f = V.validate_index(bad, NT)
        want = V.FLAG_INDEX_RANGE if name.startswith("range") else V.FLAG_INDEX_ORDER
        assert f & want, (name, f)


def test_validate_finite_flags(V, case):
    pre, path, q, k, v, o = case
    assert V.validate_finite(q) == 0
    for val in (float("nan"), float("inf"), -float("inf")):
        x = q.clone()
        x[1, 100, 17] = val
        assert V.validate_finite(x) == V.FLAG_NONFINITE
    # a [N, Hh, d] view (token-major strides)
    x = q.transpose(0, 1).contiguous().transpose(0, 1)
    x[0, 5, 0] = float("nan")
    assert V.validate_finite(x) == V.FLAG_NONFINITE


@pytest.mark.parametrize("entry", ["tokens", "tiled"])
def test_debug_mode_returns_error_codes(V, case, entry):
    pre, path, q, k, v, o = case
    NT = path.shape.n_tiles
    prev = V.set_debug(True)
    try:
        tiled = V.SparseAttention(pre.lat, [pre.cfg], pre.heads, pre.d, path.weights, sparsity=pre.sparsity,
                                  device=q.device, mode="tiled")
        tiled(q, k, v)
        for name, (bad, code) in _bad_lists(path.idx, NT).items():
            with pytest.raises(V.VedaError, match=code):
                if entry == "tokens":
                    V.sparse_attn_fwd_tokens(q, k, v, pre.lat, [pre.cfg], bad, path.mask)
                else:
                    V.sparse_attn_fwd(tiled.qt, tiled.kt, tiled.vt, bad, tiled.mask)
        x = q.clone()
        x[0, 3, 3] = float("nan")
        with pytest.raises(V.VedaError, match="VEDA_ERR_NONFINITE"):
            if entry == "tokens":
                V.sparse_attn_fwd_tokens(x, k, v, pre.lat, [pre.cfg], path.idx, path.mask)
            else:
                V.sparse_attn_fwd(V.tile_permute(x, pre.lat, [pre.cfg], meta=False)[0], tiled.kt, tiled.vt, path.idx,
                                  tiled.mask)
        s = path.scores.clone()
        s[1, 2, 3] = float("nan")
        with pytest.raises(V.VedaError, match="VEDA_ERR_NONFINITE"):
            V.select_topk(s, path.k)
        # valid inputs pass in debug mode and give the same output
        o2 = V.sparse_attn_fwd_tokens(q, k, v, pre.lat, [pre.cfg], path.idx, path.mask)
        torch.cuda.synchronize()
        assert torch.equal(o2.view(torch.int16), o.view(torch.int16))
    finally:
        V.set_debug(prev)


def test_out_of_range_lists_stay_inside_the_head(V, case):
    """Default mode: a list with entries outside [0, n_tiles) is clamped inside the kernel --
    no fault, and every other query tile's output is unchanged."""
    pre, path, q, k, v, o = case
    NT = path.shape.n_tiles
    bad = path.idx.clone()
    bad[0, 3] = torch.tensor([NT + 1000] * path.k, dtype=torch.int32)
    bad[1, 4, 0] = -7
    o2 = V.sparse_attn_fwd_tokens(q, k, v, pre.lat, [pre.cfg], bad, path.mask)
    torch.cuda.synchronize()
    assert torch.isfinite(o2.float()).all()
    # rows of tokens outside the two corrupted query tiles are bit-identical
    o2t = V.tile_permute(o2, pre.lat, [pre.cfg], meta=False)[0]
    ot = V.tile_permute(o, pre.lat, [pre.cfg], meta=False)[0]
    keep = torch.ones(pre.heads, NT, dtype=torch.bool, device=o.device)
    keep[0, 3] = False
    keep[1, 4] = False
    assert torch.equal(o2t[keep].view(torch.int16), ot[keep].view(torch.int16))


def test_fused_select_debug_mode_flags_nonfinite_scores(V, case):
    """Debug mode checks the pooled descriptors (and every score chunk) of
    veda_tile_select_pooled: a NaN or inf descriptor gives VEDA_ERR_NONFINITE; valid inputs
    give the same lists as the default mode; k outside [1, n_tiles] is VEDA_ERR_K_RANGE."""
    pre, path, q, k, v, o = case
    with pytest.raises(V.VedaError, match="VEDA_ERR_K_RANGE"):
        V.tile_select_pooled(path.zq, path.zk, path.cnt, path.scorer, path.shape.n_tiles + 1)
    prev = V.set_debug(1)
    try:
        idx = V.tile_select_pooled(path.zq, path.zk, path.cnt, path.scorer, path.k, heads_per_chunk=1)
        torch.cuda.synchronize()
        assert torch.equal(idx, path.idx)
        for val in (float("nan"), float("inf")):
            zk = path.zk.clone()
            zk[1, 4, 7] = val
            with pytest.raises(V.VedaError, match="VEDA_ERR_NONFINITE"):
                V.tile_select_pooled(path.zq, zk, path.cnt, path.scorer, path.k, heads_per_chunk=1)
    finally:
        V.set_debug(prev)
