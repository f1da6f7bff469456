"""clock64 timeline of CTA 0 of the half-tile attention kernel (VEDA_ATTN_TRACE build):
MMA groups (t, h, slot): wait start / P ok / issued; softmax blocks per slot and quarter."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_30325_b200 import synth, veda  # noqa: E402


def main():
    lib = veda.load()
    lib.veda_dbg_set_attn_trace.argtypes = [ctypes.c_void_p]
    pre = synth.PRESETS["waver12b"]
    dev = torch.device("cuda")
    heads = [0, 1, 2, 3]
    q, k, v = synth.qkv(pre, heads=heads, device=dev)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre, heads=heads).items()}
    path = veda.SparseAttention(pre.lat, [pre.cfg], len(heads), pre.d, w, sparsity=pre.sparsity, device=dev, mode="tiled")
    path(q, k, v)
    tr = torch.zeros(16 * 128 * 8, dtype=torch.int64, device=dev)
    lib.veda_dbg_set_attn_trace(ctypes.c_void_p(tr.data_ptr()))
    veda.sparse_attn_fwd(path.qt, path.kt, path.vt, path.idx, path.mask)
    tr.zero_()
    veda.sparse_attn_fwd(path.qt, path.kt, path.vt, path.idx, path.mask)
    torch.cuda.synchronize()
    t = tr.view(16, 128, 8).cpu().numpy().astype(np.int64)
    t0 = t[t > 0].min()
    t = np.where(t > 0, t - t0, -1)
    print("MMA groups n=(t*4 + h*2 + s): wait_start, P_ok, issued | d(wait) d(issue)")
    for n in range(8, 72):
        r = t[0, n]
        print(f"  n={n:3d} t={n // 4:2d} h={(n >> 1) & 1} s={n & 1}  {r[0]:8d} {r[1]:8d} {r[2]:8d} | {r[1] - r[0]:6d} {r[2] - r[1]:6d}")
    for s in (0, 1):
        for qq in (0, 1):
            r = t[1 + 4 * s + qq, 8:100]
            print(f"slot {s} quarter {qq}: wait-for-S {np.mean(r[:, 1] - r[:, 0]):.0f}, ld+max {np.mean(r[:, 2] - r[:, 1]):.0f}, "
                  f"exp+P {np.mean(r[:, 3] - r[:, 2]):.0f}, loop {np.mean(r[1:, 0] - r[:-1, 3]):.0f}, period/block {np.mean(np.diff(r[:, 1])):.0f}")
        r = t[1 + 4 * s, 8:24]
        for b in range(16):
            print(f"   slot {s} block {b + 8}: {r[b, 0]:8d} {r[b, 1]:8d} {r[b, 2]:8d} {r[b, 3]:8d}")


if __name__ == "__main__":
    main()
