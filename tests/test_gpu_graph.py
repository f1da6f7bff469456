"""SparseAttention.capture: one call recorded into a CUDA graph (pool -> fused score + top-k
with its side-stream fork / join -> attention) replays bit-identically to the eager call, and
reads its input buffers live (new contents of q, k, v give the new call's result)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("preset,heads", [("wan1.3b", 12), ("waver12b", 3)])
def test_graph_replay_bit_identical(preset, heads):
    from paper_2605_30325_b200 import build, synth, veda

    build.build()
    veda.load()
    pre = synth.PRESETS[preset]
    dev = torch.device("cuda", 0)
    hs = list(range(heads))
    q, k, v = synth.qkv(pre, heads=hs, device=dev)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre, heads=hs).items()}
    path = veda.SparseAttention(pre.lat, [pre.cfg], heads, pre.d, w, sparsity=pre.sparsity, device=dev)
    out = torch.empty_like(q)
    path(q, k, v, out=out)
    torch.cuda.synchronize()
    want, want_idx = out.clone(), path.idx.clone()

    g = path.capture(q, k, v, out)
    out.zero_()
    path.idx.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, want)
    assert torch.equal(path.idx, want_idx)

    # live inputs: swap q and k contents, replay, compare with an eager call on the same data
    qs, ks = q.clone(), k.clone()
    q.copy_(ks)
    k.copy_(qs)
    g.replay()
    torch.cuda.synchronize()
    got = out.clone()
    path(q, k, v, out=out)
    torch.cuda.synchronize()
    assert torch.equal(got, out)
    assert not torch.equal(got, want)
