"""clock64 timeline of CTA 0 of the P-in-shared-memory attention schedule (VEDA_ATTN=ps,
VEDA_ATTN_TRACE build; see tools/attn_hs_trace.py for the build line).
MMA fields per kept tile t: 0 step start, 1 both QK(t+1) issued, 2/3 P_FULL(slot 0/1) ok,
4/5 V stage of slot 0/1 ready.  Softmax fields: 0 wait-S start, 1 S ok, 2 S loaded + freed,
3 max done + P buffer free, 4 exps + P stores done, 5 P_FULL arrived.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import synth, veda  # noqa: E402


def main():
    lib = veda.load()
    lib.veda_dbg_set_attn_trace.argtypes = [ctypes.c_void_p]
    pre = synth.PRESETS["waver12b"]
    dev = torch.device("cuda")
    heads = [0, 1]
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
    lo, hi = 8, 90
    m = t[0, lo:hi]
    print("MMA per tile (mean clk): S_FREE+ring waits+2 QK", np.mean(m[:, 1] - m[:, 0]).round(),
          "| P_FULL(0) wait", np.mean(m[:, 2] - m[:, 1]).round(), "| V(0) wait", np.mean(m[:, 4] - m[:, 2]).round(),
          "| PV0 + P_FULL(1)", np.mean(m[:, 3] - m[:, 4]).round(), "| V(1) wait", np.mean(m[:, 5] - m[:, 3]).round(),
          "| period", np.mean(np.diff(m[:, 0])).round())
    names = ["wait S", "ld+free", "max+Pbuf", "exp+st", "arrive"]
    for s in (0, 1):
        for qq in range(4):
            r = t[1 + 4 * s + qq, lo:hi]
            d = [np.mean(r[:, i + 1] - r[:, i]) for i in range(5)]
            print(f"slot {s} q{qq}: " + ", ".join(f"{n} {x:.0f}" for n, x in zip(names, d)) +
                  f" | period {np.mean(np.diff(r[:, 1])):.0f}")
    print("steps (MMA fields 0..5 | slot0 q0 fields 0..5 | slot1 q0 fields 0..5)")
    for n in range(lo, lo + 12):
        print(f"{n:3d} " + " ".join(f"{x:7d}" for x in t[0, n, :6]) + " | " + " ".join(f"{x:7d}" for x in t[1, n, :6]) +
              " | " + " ".join(f"{x:7d}" for x in t[5, n, :6]))


if __name__ == "__main__":
    main()
