"""Sparsity x sequence-length sweep of the full path on one B200.

For each workload (latent shape, heads) and sparsity: ms per call of the whole path
(a1-a7), the attention kernel alone, executed TFLOP/s, and the same attention kernel run
dense (k = N_T; timed once per workload) -> speedup vs dense.  Writes JSON + markdown.

    python tools/sweep.py [--out profiles/r01_sweep] [--workloads wan1.3b,wan14b,waver12b,...]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import synth, veda  # noqa: E402

# SURVEY.md §8(d) d2 shapes (24 heads, d = 128, tile (4,4,8)) plus the three model presets
SHAPES = {
    "wan1.3b": ((21, 30, 52), 12),
    "waver480p121f": ((31, 30, 54), 24),   # 50,220 tokens
    "wan14b": ((21, 45, 80), 40),
    "waver720p121f": ((31, 45, 80), 24),   # Fig. 7 shape
    "waver12b": ((61, 45, 80), 24),
}
SPARSITIES = (0.80, 0.90, 0.95, 0.98)


def timeit(fn, reps):
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
    ap.add_argument("--out", default="profiles/r01_sweep")
    ap.add_argument("--workloads", default=",".join(SHAPES))
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    veda.load()
    dev = torch.device("cuda")
    rows = []
    for name in a.workloads.split(","):
        lat, heads = SHAPES[name]
        pre = synth.Preset(name, lat, heads, 128, (4, 4, 8), 0.95)
        q, k, v = synth.qkv(pre, device=dev)
        w = {n: t.to(dev) for n, t in synth.scorer_weights(pre).items()}
        out = torch.empty_like(q)
        dense_ms = None
        for sp in SPARSITIES:
            path = veda.SparseAttention(lat, [pre.cfg], heads, 128, w, sparsity=sp, device=dev, mode="tiled")
            NT, B = path.shape.n_tiles, path.shape.B
            call_ms = timeit(lambda: path(q, k, v, out=out), a.reps)
            attn_ms = timeit(lambda: veda.sparse_attn_fwd(path.qt, path.kt, path.vt, path.idx, path.mask, out=path.ot),
                             a.reps)
            if dense_ms is None:
                idx_d = torch.arange(NT, dtype=torch.int32, device=dev).expand(heads, NT, NT).contiguous()
                dense_ms = timeit(lambda: veda.sparse_attn_fwd(path.qt, path.kt, path.vt, idx_d, path.mask,
                                                               out=path.ot), 1)
                dense_tf = 4.0 * B * B * 128 * NT * NT * heads / dense_ms / 1e9
                del idx_d
            tf = 4.0 * B * B * 128 * path.k * NT * heads / attn_ms / 1e9
            r = dict(workload=name, latent=list(lat), tokens=lat[0] * lat[1] * lat[2], heads=heads, n_tiles=NT,
                     sparsity=sp, k=path.k, call_ms=round(call_ms, 3), attn_ms=round(attn_ms, 3),
                     attn_tflops=round(tf, 1), dense_attn_ms=round(dense_ms, 2), dense_tflops=round(dense_tf, 1),
                     speedup_call_vs_dense_kernel=round(dense_ms / call_ms, 2))
            rows.append(r)
            print(json.dumps(r), flush=True)
            del path
        del q, k, v, w, out
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(rows, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as f:
        f.write("| workload | tokens | heads | N_T | sparsity | k | call ms | attn ms | attn TFLOP/s | dense attn ms | "
                "dense TFLOP/s | call speedup vs dense |\n|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|\n")
        for r in rows:
            f.write(f"| {r['workload']} | {r['tokens']} | {r['heads']} | {r['n_tiles']} | {r['sparsity']:.2f} | "
                    f"{r['k']} | {r['call_ms']} | {r['attn_ms']} | {r['attn_tflops']} | {r['dense_attn_ms']} | "
                    f"{r['dense_tflops']} | {r['speedup_call_vs_dense_kernel']} |\n")


if __name__ == "__main__":
    main()
