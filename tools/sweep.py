"""Sparsity x sequence-length sweep of the full path on one B200.

For each workload (latent shape, heads) and sparsity: ms per call of the whole path
(a1-a7, token-layout form), the attention kernel alone (incl. the fused untiling),
executed TFLOP/s, and the same attention kernel run dense (k = N_T, i.e. 0 % sparsity;
timed once per workload) -> speedup vs dense.  With --shards, also the call time of the
busiest rank of a G-way head-sharded run (ceil(Hh/G) heads; the path has no collective,
so this is the rank-local work) -- measured on ONE B200, not a multi-GPU measurement;
where G does not divide the head count, also the busiest rank of the (head x query tile)
unit shares (shard.unit_range, veda_sparse_attn_fwd_tokens_units).
Writes JSON + markdown.

    python tools/sweep.py [--out profiles/r01_sweep] [--workloads wan1.3b,wan14b,waver12b,...]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import shard, synth, veda  # noqa: E402

# SURVEY.md §8(d) d2 shapes (24 heads, d = 128, tile (4,4,8)) plus the three model presets
SHAPES = {
    "wan1.3b": ((21, 30, 52), 12),
    "waver480p121f": ((31, 30, 54), 24),   # 50,220 tokens
    "wan14b": ((21, 45, 80), 40),
    "waver720p121f": ((31, 45, 80), 24),   # Fig. 7 shape
    "waver12b": ((61, 45, 80), 24),
}
SPARSITIES = (0.80, 0.90, 0.95, 0.98)
SHARDS = (2, 4, 8)


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
    ap.add_argument("--shards", action="store_true", help="also time the busiest rank of 2/4/8-way head sharding")
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
            path = veda.SparseAttention(lat, [pre.cfg], heads, 128, w, sparsity=sp, device=dev)
            NT, B = path.shape.n_tiles, path.shape.B
            call_ms = timeit(lambda: path(q, k, v, out=out), a.reps)
            attn_ms = timeit(lambda: veda.sparse_attn_fwd_tokens(q, k, v, lat, [pre.cfg], path.idx, path.mask,
                                                                 out=out), a.reps)
            if dense_ms is None:
                idx_d = torch.arange(NT, dtype=torch.int32, device=dev).expand(heads, NT, NT).contiguous()
                dense_ms = timeit(lambda: veda.sparse_attn_fwd_tokens(q, k, v, lat, [pre.cfg], idx_d, path.mask,
                                                                      out=out), 1)
                dense_tf = 4.0 * B * B * 128 * NT * NT * heads / dense_ms / 1e9
                del idx_d
            tf = 4.0 * B * B * 128 * path.k * NT * heads / attn_ms / 1e9
            r = dict(workload=name, latent=list(lat), tokens=lat[0] * lat[1] * lat[2], heads=heads, n_tiles=NT,
                     sparsity=sp, k=path.k, call_ms=round(call_ms, 3), attn_ms=round(attn_ms, 3),
                     attn_tflops=round(tf, 1), dense_attn_ms=round(dense_ms, 2), dense_tflops=round(dense_tf, 1),
                     speedup_call_vs_dense_kernel=round(dense_ms / call_ms, 2))
            del path
            if a.shards:
                for G in SHARDS:
                    hr = -(-heads // G)
                    wr = {n: t[:hr] for n, t in w.items()}
                    pr = veda.SparseAttention(lat, [pre.cfg], hr, 128, wr, sparsity=sp, device=dev)
                    r[f"rank_ms_G{G}"] = round(timeit(lambda: pr(q[:hr], k[:hr], v[:hr], out=out[:hr]), a.reps), 3)
                    del pr
                    if heads % G:  # unit shares (shard.unit_range): the busiest rank over all G
                        worst = 0.0
                        for rk in range(G):
                            u = shard.unit_range(heads, NT, rk, G)
                            pr = veda.SparseAttention(lat, [pre.cfg], heads, 128, w, sparsity=sp, device=dev,
                                                      units=(u.start, u.stop))
                            worst = max(worst, timeit(lambda: pr(q, k, v, out=out), a.reps))
                            del pr
                        r[f"rank_ms_G{G}_units"] = round(worst, 3)
            rows.append(r)
            print(json.dumps(r), flush=True)
        del q, k, v, w, out
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(rows, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as f:
        gs = [G for G in SHARDS if rows and f"rank_ms_G{G}" in rows[0]]
        f.write("| workload | tokens | heads | N_T | sparsity | k | call ms | attn ms | attn TFLOP/s | dense attn ms | "
                "dense TFLOP/s | call speedup vs dense |" + "".join(f" busiest rank, G={G} (ms, 1-GPU proxy) |" for G in gs) +
                "\n|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|" + "---:|" * len(gs) + "\n")
        for r in rows:
            f.write(f"| {r['workload']} | {r['tokens']} | {r['heads']} | {r['n_tiles']} | {r['sparsity']:.2f} | "
                    f"{r['k']} | {r['call_ms']} | {r['attn_ms']} | {r['attn_tflops']} | {r['dense_attn_ms']} | "
                    f"{r['dense_tflops']} | {r['speedup_call_vs_dense_kernel']} |" +
                    "".join(f" {r[f'rank_ms_G{G}']}" + (f" (units: {r[f'rank_ms_G{G}_units']})"
                                                        if f"rank_ms_G{G}_units" in r else "") + " |" for G in gs) +
                    "\n")


if __name__ == "__main__":
    main()
