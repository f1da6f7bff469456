"""Score + top-k: the two-call form (tile_score_pooled -> select_topk, a full [Hh, N_T, N_T]
score tensor) against veda_tile_select_pooled at several head-chunk sizes.

    python tools/select_bench.py [--workload waver12b]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import synth, veda  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="waver12b")
    ap.add_argument("--chunks", default="1,2,3,4,6,8,12,24")
    a = ap.parse_args()
    veda.load()
    pre = synth.PRESETS[a.workload]
    dev = torch.device("cuda")
    q, k, v = synth.qkv(pre, device=dev)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre).items()}
    path = veda.SparseAttention(pre.lat, [pre.cfg], pre.heads, pre.d, w, sparsity=pre.sparsity, keep_scores=True)
    path(q, k, v)
    ref = path.idx.clone()
    t2 = timeit(lambda: (veda.tile_score_pooled(path.zq, path.zk, path.cnt, path.scorer, path.ws, path.scores),
                         veda.select_topk(path.scores, path.k, path.idx)))
    print(f"{a.workload}: two calls (full S, {path.scores.numel() * 4 / 1e6:.0f} MB): {t2:.3f} ms", flush=True)
    out = torch.empty_like(ref)
    for hpc in [int(x) for x in a.chunks.split(",") if int(x) <= pre.heads]:
        ws = veda.SelectWorkspace(pre.heads, path.shape.n_tiles, pre.d, path.scorer, dev, hpc)
        t = timeit(lambda: veda.tile_select_pooled(path.zq, path.zk, path.cnt, path.scorer, path.k, hpc, ws, out))
        same = torch.equal(out, ref)
        print(f"  select, {hpc:2d} heads per chunk ({hpc * path.shape.n_tiles ** 2 * 4 / 1e6:6.1f} MB): {t:.3f} ms"
              f"  lists {'identical' if same else 'DIFFER'}", flush=True)


if __name__ == "__main__":
    main()
