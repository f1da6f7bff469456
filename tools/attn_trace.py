"""Per-step clock64 timeline of CTA 0 of the attention kernel (VEDA_ATTN_TRACE build).

    VEDA_LIB=paper_2605_30325_b200/libveda_trace.so python tools/attn_trace.py [--heads 2]
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
    ap.add_argument("--heads", type=int, default=2)
    ap.add_argument("--steps", type=int, default=24)
    ap.add_argument("--sparsity", type=float, default=None)
    a = ap.parse_args()
    lib = veda.load()
    lib.veda_dbg_set_attn_trace.argtypes = [ctypes.c_void_p]
    pre = synth.PRESETS["waver12b"]
    if a.sparsity is not None:
        pre = synth.Preset(pre.name, pre.lat, pre.heads, pre.d, pre.cfg, a.sparsity)
    dev = torch.device("cuda")
    heads = list(range(a.heads))
    q, k, v = synth.qkv(pre, heads=heads, device=dev)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre, heads=heads).items()}
    path = veda.SparseAttention(pre.lat, [pre.cfg], len(heads), pre.d, w, sparsity=pre.sparsity, device=dev, mode="tiled")
    path(q, k, v)
    tr = torch.zeros(16 * 128 * 8, dtype=torch.int64, device=dev)
    lib.veda_dbg_set_attn_trace(ctypes.c_void_p(tr.data_ptr()))
    veda.sparse_attn_fwd(path.qt, path.kt, path.vt, path.idx, path.mask)  # warm
    tr.zero_()
    veda.sparse_attn_fwd(path.qt, path.kt, path.vt, path.idx, path.mask)
    torch.cuda.synchronize()
    t = tr.view(16, 128, 8).cpu().numpy().astype(np.int64)
    t0 = t[t > 0].min()
    t = np.where(t > 0, t - t0, -1)
    for role, name in ((0, "thread (both slots)"),):
        print(f"MMA warp {name}: qk[n]: wait_ring_start, ring_ok, issued | pv[n]: wait_P_start, P_ok, issued")
        for n in range(a.steps):
            print(f"  n={n:3d} qk {t[role, n, 0]:8d} {t[role, n, 1]:8d} {t[role, n, 2]:8d} | "
                  f"pv {t[role, n, 3]:8d} {t[role, n, 4]:8d} {t[role, n, 5]:8d}")
    for s in (0, 1):
        for qq in range(4):
            r = t[1 + 4 * s + qq, 4:a.steps]
            print(f"slot {s} quarter {qq}: wait-for-S {np.mean(r[:, 1] - r[:, 0]):.0f}, ld {np.mean(r[:, 2] - r[:, 1]):.0f}, "
                  f"max {np.mean(r[:, 3] - r[:, 2]):.0f}, exp+st {np.mean(r[:, 4] - r[:, 3]):.0f}, "
                  f"P_arrive - S_ok {np.mean(r[:, 5] - r[:, 1]):.0f}, P_arrive rel. to quarter 0 "
                  f"{np.mean(r[:, 5] - t[1 + 4 * s, 4:a.steps, 5]):.0f}")
    for s in (0, 1):
        print(f"slot {s} softmax (warp lane 0): wait_S_start, S_ok, ld_done, max_done, exp_st_done, P_arrive | "
              "dS_wait dLd dMax dExp dArr")
        for n in range(a.steps):
            r = t[1 + 4 * s, n]
            d = [r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], r[5] - r[4]]
            print(f"  t={n:3d} {r[0]:8d} {r[1]:8d} {r[2]:8d} {r[3]:8d} {r[4]:8d} {r[5]:8d} | " + " ".join(f"{x:6d}" for x in d))
    for s in (0, 1):
        for qq in range(4):
            r = t[1 + 4 * s + qq, 1:a.steps]
            print(f"slot {s} quarter {qq}: rescaled tiles {np.mean(r[:, 6] >= 0):.3f} (after the first)")
    # steady-state averages
    for s in (0, 1):
        r = t[1 + 4 * s, 4:a.steps]
        per = np.diff(r[:, 1]).mean()
        print(f"slot {s}: mean period between S arrivals {per:.0f} clk; mean wait-for-S {np.mean(r[:, 1] - r[:, 0]):.0f}, "
              f"ld {np.mean(r[:, 2] - r[:, 1]):.0f}, max {np.mean(r[:, 3] - r[:, 2]):.0f}, exp+st {np.mean(r[:, 4] - r[:, 3]):.0f}, "
              f"arrive {np.mean(r[:, 5] - r[:, 4]):.0f}")


if __name__ == "__main__":
    main()
