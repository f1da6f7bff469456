"""Time veda_sparse_attn_fwd alone on a Waver-shaped problem (for kernel A/B experiments).

    VEDA_LIB=... python tools/attn_bench.py [--heads 8] [--reps 10] [--regime path|random|dense]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import synth, veda  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--regime", default="path")
    ap.add_argument("--workload", default="waver12b")
    ap.add_argument("--sparsity", type=float, default=None, help="override the workload's sparsity")
    ap.add_argument("--tokens", action="store_true", help="time the token-layout kernel (the path's) instead")
    a = ap.parse_args()
    veda.load()
    pre = synth.PRESETS[a.workload]
    dev = torch.device("cuda")
    heads = list(range(a.heads))
    q, k, v = synth.qkv(pre, heads=heads, device=dev)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre, heads=heads).items()}
    path = veda.SparseAttention(pre.lat, [pre.cfg], len(heads), pre.d, w, sparsity=pre.sparsity if a.sparsity is None else a.sparsity, device=dev, mode="tiled")
    path(q, k, v)
    NT, B, kk = path.shape.n_tiles, path.shape.B, path.k
    if a.regime == "random":
        idx = synth.random_index_lists(len(heads), NT, kk).to(dev)
    elif a.regime == "dense":
        idx = torch.arange(NT, dtype=torch.int32, device=dev).expand(len(heads), NT, NT).contiguous()
        kk = NT
    else:
        idx = path.idx
    if a.tokens:
        out = torch.empty_like(q)
        run = lambda: veda.sparse_attn_fwd_tokens(q, k, v, pre.lat, [pre.cfg], idx, path.mask, out=out)
    else:
        out = torch.empty_like(path.ot)
        run = lambda: veda.sparse_attn_fwd(path.qt, path.kt, path.vt, idx, path.mask, out=out)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    flops = 4.0 * B * B * pre.d * kk * NT * len(heads)
    print(f"{os.environ.get('VEDA_LIB', 'libveda.so').split('/')[-1]:28s} {a.regime:6s} heads={a.heads} "
          f"{'tokens' if a.tokens else 'tiled'} k={kk} "
          f"{ms:8.3f} ms  {flops / ms / 1e9:7.1f} TFLOP/s", flush=True)
    return out


if __name__ == "__main__":
    main()
