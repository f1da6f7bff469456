"""Head-aware tiling search (Alg. 1) at a preset's full shape on synthetic heads:
time per calibration sample, per candidate, and the chosen pi* per head.

python tools/search_bench.py [--preset waver12b] [--heads 4] [--k-top 96]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import build, search, synth, veda  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="waver12b")
    ap.add_argument("--heads", type=int, default=4)
    ap.add_argument("--k-top", type=int, default=96)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    build.build()
    pre = synth.PRESETS[a.preset]
    dev = torch.device("cuda")
    q, k, v = synth.qkv(pre, heads=range(a.heads), device=dev)
    ts = search.TilingSearch(pre.lat, a.heads, pre.d, k_top=a.k_top, B=128)
    # warm-up on one candidate (module load, tensor maps, allocator)
    o_fu, lse = ts.full_attention(q, k, v)
    ts.candidate(q, k, v, lse, ts.cands[0])
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(ts.cands) + 2)]
    t0 = time.time()
    ev[0].record()
    o_fu, lse = ts.full_attention(q, k, v)
    ev[1].record()
    per = []
    for c, cfg in enumerate(ts.cands):
        o_sp, _ = ts.candidate(q, k, v, lse, cfg)
        veda.sq_err(o_fu, o_sp, ts.err[c])
        ev[c + 2].record()
    torch.cuda.synchronize()
    wall = time.time() - t0
    E = ts.errors()
    res = {
        "preset": a.preset, "heads": a.heads, "k_top": a.k_top, "candidates": len(ts.cands),
        "dense_pass_ms": ev[0].elapsed_time(ev[1]),
        "search_ms": ev[0].elapsed_time(ev[-1]), "wall_s": wall,
        "per_candidate_ms": {str(cfg): round(ev[c + 1].elapsed_time(ev[c + 2]), 2) for c, cfg in enumerate(ts.cands)},
        "n_tiles": {str(cfg): veda.tiled_shape(pre.lat, [cfg], 1).n_tiles for cfg in ts.cands},
        "best": [list(b) for b in ts.best()],
        "rel_err_best": [float(E[h].min() / E[h].max()) for h in range(a.heads)],
        "E": {str(cfg): [float(x) for x in E[:, c]] for c, cfg in enumerate(ts.cands)},
    }
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
