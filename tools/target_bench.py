"""Time the oracle-mask passes at the Waver-12B shape: dense lse pass (veda_sparse_attn_fwd,
k = N_T), veda_target_scores (QK^T only), top-k on S_tgt, and the recall of the path's
predicted lists (random-init scorer) against the oracle mask.

python tools/target_bench.py [--heads 24] [--iters 5]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import build, synth, veda  # noqa: E402


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=24)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--preset", default="waver12b")
    a = ap.parse_args()
    build.build()
    pre = synth.PRESETS[a.preset]
    dev = torch.device("cuda")
    q, k, v = synth.qkv(pre, heads=range(a.heads), device=dev)
    w = {n: t[:a.heads].contiguous().to(dev) for n, t in synth.scorer_weights(pre).items()}
    path = veda.SparseAttention(pre.lat, [pre.cfg], a.heads, pre.d, w, sparsity=pre.sparsity, mode="tiled")
    path(q, k, v)
    qt, kt, vt, mask, cnt = path.qt, path.kt, path.vt, path.mask, path.cnt
    Hh, NT, B, d = qt.shape
    dense = torch.arange(NT, dtype=torch.int32, device=dev).expand(Hh, NT, NT).contiguous()
    out = torch.empty_like(qt)
    lse = torch.empty((Hh, NT, B), dtype=torch.float32, device=dev)
    s_tgt = torch.empty((Hh, NT, NT), dtype=torch.float32, device=dev)
    idx_star = torch.empty((Hh, NT, path.k), dtype=torch.int32, device=dev)
    rec = torch.empty((), dtype=torch.float64, device=dev)

    def lse_pass():
        _check(veda.load().veda_sparse_attn_fwd(veda._ptr(qt), veda._ptr(kt), veda._ptr(vt), veda._ptr(dense),
                                                veda._ptr(mask), Hh, NT, B, d, NT, 0.0, veda._ptr(out),
                                                veda._ptr(lse), veda._stream()))

    def _check(st):
        if st:
            raise RuntimeError(veda.load().veda_last_error().decode())

    t_lse = timed(lse_pass, a.iters)
    t_tgt = timed(lambda: veda.target_scores(qt, kt, mask, lse, out=s_tgt), a.iters)
    t_topk = timed(lambda: veda.select_topk(s_tgt, path.k, out=idx_star), a.iters)
    t_rec = timed(lambda: veda.tile_recall(path.idx, idx_star, cnt, out=rec), a.iters)
    flop_qk = 2.0 * B * B * d * NT * NT * Hh
    res = {
        "preset": a.preset, "heads": Hh, "n_tiles": NT, "k": path.k,
        "lse_pass_ms": t_lse, "lse_pass_tflops": 2 * flop_qk / t_lse / 1e9,
        "target_ms": t_tgt, "target_tflops": flop_qk / t_tgt / 1e9,
        "topk_ms": t_topk, "recall_ms": t_rec,
        "recall_pred_vs_oracle_mask": rec.item(),
        "recall_random_expected": path.k / NT,
    }
    print(json.dumps(res))


if __name__ == "__main__":
    main()
