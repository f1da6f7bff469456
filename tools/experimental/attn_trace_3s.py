"""Per-step clock64 timeline of CTA 0 of the attention kernel (VEDA_ATTN_TRACE build).

    VEDA_NVCC_EXTRA=-DVEDA_ATTN_TRACE VEDA_LIB_OUT=paper_2605_30325_b200/libveda_trace.so \
        VEDA_BUILD_TAG=_trace python -m paper_2605_30325_b200.build --force
    VEDA_LIB=paper_2605_30325_b200/libveda_trace.so python tools/attn_trace.py [--heads 4]

Stamps (csrc/attn_fwd.cu TR): MMA thread, per tile g: PV wait start (0), P ok (4), V ok (1),
QK(g) wait start (2), K ok (3).  Softmax warp (set s, quarter q), per tile of the set:
S wait start (0), S ok (1), max done (2), reference max in (3), exp + P stores done (4),
P_FULL arrive (5).
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import synth, veda  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=4)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--workload", default="waver12b")
    a = ap.parse_args()
    lib = veda.load()
    lib.veda_dbg_set_attn_trace.argtypes = [ctypes.c_void_p]
    pre = synth.PRESETS[a.workload]
    dev = torch.device("cuda")
    heads = list(range(a.heads))
    q, k, v = synth.qkv(pre, heads=heads, device=dev)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre, heads=heads).items()}
    path = veda.SparseAttention(pre.lat, [pre.cfg], len(heads), pre.d, w, sparsity=pre.sparsity, device=dev)
    path(q, k, v)
    tr = torch.zeros(16 * 128 * 8, dtype=torch.int64, device=dev)
    lib.veda_dbg_set_attn_trace(ctypes.c_void_p(tr.data_ptr()))
    out = torch.empty_like(q)
    run = lambda: veda.sparse_attn_fwd_tokens(q, k, v, pre.lat, [pre.cfg], path.idx, path.mask, out=out)
    run()
    tr.zero_()
    run()
    torch.cuda.synchronize()
    t = tr.view(16, 128, 8).cpu().numpy().astype(np.int64)
    t0 = t[t > 0].min()
    t = np.where(t > 0, t - t0, -1)
    S = a.steps
    print("MMA: g | PV: wait0  P_ok  V_ok | QK(g): wait0 K_ok")
    for g in range(S):
        r = t[0, g]
        print(f"  g={g:3d} PV {r[0]:8d} {r[4]:8d} {r[1]:8d} | QK {r[2]:8d} {r[3]:8d}")
    pv_ok = t[0, 8:S, 1]
    print(f"MMA: mean PV-to-PV period {np.diff(pv_ok).mean():.0f} clk; mean wait for P "
          f"{np.mean(t[0, 8:S, 4] - t[0, 8:S, 0]):.0f}, for V {np.mean(t[0, 8:S, 1] - t[0, 8:S, 4]):.0f}, "
          f"for K {np.mean(t[0, 8:S, 3] - t[0, 8:S, 2]):.0f}")
    for s in (0, 1):
        for qq in range(4):
            r = t[1 + 4 * s + qq, 4:S // 2]
            print(f"set {s} quarter {qq}: wait-S {np.mean(r[:, 1] - r[:, 0]):.0f}, ld+max {np.mean(r[:, 2] - r[:, 1]):.0f}, "
                  f"mbox {np.mean(r[:, 3] - r[:, 2]):.0f} (get {np.mean(r[:, 6] - r[:, 2]):.0f}, vote {np.mean(r[:, 7] - r[:, 6]):.0f}, put {np.mean(r[:, 3] - r[:, 7]):.0f}), exp+st {np.mean(r[:, 4] - r[:, 3]):.0f}, "
                  f"arrive {np.mean(r[:, 5] - r[:, 4]):.0f}, S_ok->P {np.mean(r[:, 5] - r[:, 1]):.0f}")
    print("per tile g: S_ok of quarters 0-3 | P arrive of quarters 0-3 | MMA P_ok")
    for g in range(8, S):
        s, n = g % 2, g // 2
        r = t[1 + 4 * s:5 + 4 * s, n]
        print(f"  g={g:3d} S_ok " + " ".join(f"{x:8d}" for x in r[:, 1]) + " | P " + " ".join(f"{x:8d}" for x in r[:, 5])
              + f" | {t[0, g, 4]:8d}  (P spread {r[:, 5].max() - r[:, 5].min()}, S_ok spread {r[:, 1].max() - r[:, 1].min()})")
    print("reference-max hand-off, quarter 0: g | publish(g-1) by the other set | max done(g) | get done(g)")
    for g in range(8, min(S, 30)):
        a = t[1 + 4 * ((g - 1) % 2), (g - 1) // 2, 3]
        b = t[1 + 4 * (g % 2), g // 2, 2]
        c = t[1 + 4 * (g % 2), g // 2, 6]
        print(f"  g={g:3d} {a:8d} {b:8d} {c:8d}   get-after-publish {c - a:6d}, get-after-max {c - b:6d}")
    np.save("gpurun_out/trace_raw.npy", t)
    for s in (0, 1):
        print(f"set {s} quarter 0 per tile: S_wait0 S_ok max mbox exp P")
        for n in range(S // 2):
            r = t[1 + 4 * s, n]
            print(f"  n={n:3d} " + " ".join(f"{x:8d}" for x in r[:6]))


if __name__ == "__main__":
    main()
