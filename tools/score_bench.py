"""Time the scoring sub-steps (TripPool, phi layers, pair scores, top-k) on a preset."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import synth, veda  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main(name="waver12b"):
    veda.load()
    pre = synth.PRESETS[name]
    dev = torch.device("cuda")
    q, k, v = synth.qkv(pre, device=dev)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre).items()}
    path = veda.SparseAttention(pre.lat, [pre.cfg], pre.heads, pre.d, w, sparsity=pre.sparsity, device=dev, mode="tiled")
    path(q, k, v)
    Hh, NT = pre.heads, path.shape.n_tiles
    din, dh, dl = 3 * pre.d, w["w1q"].shape[-1], w["w2q"].shape[-1]
    z = veda.trippool(path.qt, path.mask)
    e = veda.project(z, w["w1q"], w["b1q"], w["w2q"], w["b2q"])
    t_pool = timeit(lambda: veda.trippool(path.qt, path.mask))
    t_proj = timeit(lambda: veda.project(z, w["w1q"], w["b1q"], w["w2q"], w["b2q"]))
    t_pair = timeit(lambda: veda.pair_scores(e, e, path.cnt))
    t_score = timeit(lambda: veda.tile_score(path.qt, path.kt, path.cnt, path.mask, path.scorer, path.ws, path.scores))
    t_topk = timeit(lambda: veda.select_topk(path.scores, path.k, path.idx))
    f_proj = 2.0 * Hh * NT * (din * dh + dh * dl)
    f_pair = 2.0 * Hh * NT * NT * dl
    print(f"{name}: trippool {t_pool:.3f} ms ({2*Hh*NT*128*pre.d*2/t_pool/1e6:.0f} GB/s) | "
          f"project {t_proj:.3f} ms ({f_proj/t_proj/1e9:.1f} TFLOP/s fp64) | pair_scores {t_pair:.3f} ms "
          f"({f_pair/t_pair/1e9:.1f} TFLOP/s) | tile_score total {t_score:.3f} ms | topk {t_topk:.3f} ms")


if __name__ == "__main__":
    main(*sys.argv[1:])
