"""Time veda_select_topk alone on the path's own scores (Waver shape by default) and check it
against torch's sort-based reference of the same contract (S desc, then index asc).

    python tools/topk_bench.py [--workload waver12b] [--heads 24] [--reps 20]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import synth, veda  # noqa: E402


def reference(scores, k):
    s = scores.clone()
    s[s == 0] = 0.0  # -0 == +0
    n = s.shape[-1]
    # stable descending order: sort by (-S, j)
    order = torch.sort(-s, dim=-1, stable=True).indices[..., :k]
    return torch.sort(order, dim=-1).values.to(torch.int32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="waver12b")
    ap.add_argument("--heads", type=int, default=24)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    veda.load()
    pre = synth.PRESETS[a.workload]
    dev = torch.device("cuda")
    heads = list(range(a.heads))
    q, k, v = synth.qkv(pre, heads=heads, device=dev)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre, heads=heads).items()}
    path = veda.SparseAttention(pre.lat, [pre.cfg], len(heads), pre.d, w, sparsity=pre.sparsity, device=dev)
    path(q, k, v)
    S = path.scores
    kk = path.k
    out = torch.empty(S.shape[:-1] + (kk,), dtype=torch.int32, device=dev)
    veda.select_topk(S, kk, out=out)
    torch.cuda.synchronize()
    ref = torch.cat([reference(S[h:h + 1], kk) for h in range(S.shape[0])])
    bad = (out != ref).any(-1).sum().item()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        veda.select_topk(S, kk, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    nbytes = S.numel() * 4 + out.numel() * 4
    print(f"select_topk {a.workload} heads={a.heads} rows={S.shape[0] * S.shape[1]} n_tiles={S.shape[-1]} k={kk}: "
          f"{ms * 1e3:.1f} us, {nbytes / ms / 1e6:.0f} GB/s, rows differing from the sort reference: {bad}")
    fb, tr, cm = filter_stats(S, kk)
    print(f"  candidate filter (emulated): fallback rows {fb * 100:.2f} %, mean tries {tr:.2f}, mean candidates {cm:.0f}")



def filter_stats(S, k, cl=16):
    """Emulate the candidate filter's threshold search (topk.cu) in torch: fraction of rows
    that fall back to the full search, and the candidate counts."""
    import math
    x = S.reshape(-1, S.shape[-1]).double()
    fin = torch.isfinite(x)
    nf = fin.sum(-1).double()
    xs = torch.where(fin, x, torch.zeros_like(x))
    mu = xs.sum(-1) / nf
    sd = ((xs * xs).sum(-1) / nf - mu * mu).clamp_min(0).sqrt()
    want = torch.minimum(1.5 * k + 32 + 0 * nf, 0.5 * nf)
    p = want / nf
    t = torch.sqrt(-2 * torch.log(p))
    z = t - (2.515517 + t * (0.802853 + t * 0.010328)) / (1 + t * (1.432788 + t * (0.189269 + t * 0.001308)))
    ok = torch.zeros(x.shape[0], dtype=torch.bool, device=x.device)
    tries = torch.zeros_like(ok, dtype=torch.int32)
    cnt = torch.zeros(x.shape[0], device=x.device)
    lane = torch.arange(x.shape[-1], device=x.device) % 32
    for it in range(4):
        T0 = mu + z * sd
        ge = (x >= T0[:, None]) & ~ok[:, None]
        c = ge.sum(-1)
        cmax = torch.zeros(x.shape[0], 32, device=x.device, dtype=torch.long).index_add_(1, lane, ge.long()).max(-1).values
        good = (c >= k) & (cmax <= cl) & ~ok
        cnt = torch.where(good, c.double(), cnt)
        tries = torch.where(~ok, tries + 1, tries)
        ok = ok | good
        z = torch.where(c < k, z - 0.5, z + 0.3)
    return 1 - ok.double().mean().item(), tries.double().mean().item(), cnt[ok].mean().item()


if __name__ == "__main__":
    main()
