"""clock64 timeline of CTA 0 of the 1q attention schedule (VEDA_ATTN_TRACE build):

    VEDA_BUILD_TAG=_trace VEDA_LIB_OUT=paper_2605_30325_b200/libveda_trace.so \
        VEDA_NVCC_EXTRA=-DVEDA_ATTN_TRACE python -m paper_2605_30325_b200.build --force
    VEDA_ATTN=1q VEDA_LIB=paper_2605_30325_b200/libveda_trace.so python tools/attn1q_trace.py
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
    ap.add_argument("--heads", type=int, default=24)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--regime", default="path")
    a = ap.parse_args()
    lib = veda.load()
    lib.veda_dbg_set_attn1q_trace.argtypes = [ctypes.c_void_p]
    pre = synth.PRESETS["waver12b"]
    dev = torch.device("cuda")
    heads = list(range(a.heads))
    q, k, v = synth.qkv(pre, heads=heads, device=dev)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre, heads=heads).items()}
    path = veda.SparseAttention(pre.lat, [pre.cfg], len(heads), pre.d, w, sparsity=pre.sparsity, device=dev, mode="tiled")
    path(q, k, v)
    idx = path.idx
    if a.regime == "dense_seq":
        NT = path.shape.n_tiles
        idx = torch.arange(path.k, dtype=torch.int32, device=dev).expand(len(heads), NT, path.k).contiguous()
    tr = torch.zeros(4 * 256 * 8, dtype=torch.int64, device=dev)
    lib.veda_dbg_set_attn1q_trace(ctypes.c_void_p(tr.data_ptr()))
    veda.sparse_attn_fwd(path.qt, path.kt, path.vt, idx, path.mask)
    tr.zero_()
    veda.sparse_attn_fwd(path.qt, path.kt, path.vt, idx, path.mask)
    torch.cuda.synchronize()
    t = tr.view(4, 256, 8).cpu().numpy().astype(np.int64)
    t0 = t[t > 0].min()
    t = np.where(t > 0, t - t0, -1)
    print("MMA g: [start, probed, qk_waits_ok, qk_issued, P_ok, V_ok, pv_issued]")
    for g in range(a.steps):
        print(f"  g={g:3d} " + " ".join(f"{x:8d}" for x in t[0, g, :7]))
    for hf in (0, 1):
        print(f"softmax half {hf}: [wait_S, S_ok, ld+free, max+xchg, exp+st, P_arrive, rescale]")
        for g in range(a.steps):
            r = t[1 + hf, g]
            print(f"  g={g:3d} " + " ".join(f"{x:8d}" for x in r[:7]))
    print("producer: [start wait_empty, issued]")
    for n in range(a.steps):
        print(f"  L={n:3d} {t[3, n, 0]:8d} {t[3, n, 1]:8d}")
    s = t[1, 8:a.steps]
    print(f"half0 mean: period {np.diff(s[:, 1]).mean():.0f}  wait_S {np.mean(s[:, 1] - s[:, 0]):.0f}  "
          f"ld {np.mean(s[:, 2] - s[:, 1]):.0f}  max {np.mean(s[:, 3] - s[:, 2]):.0f}  "
          f"exp {np.mean(s[:, 4] - s[:, 3]):.0f}  arrive {np.mean(s[:, 5] - s[:, 4]):.0f}")
    m = t[0, 8:a.steps]
    d = np.diff(m[:, :7], axis=1).mean(axis=0)
    print("MMA mean per iteration: probe {:.0f}  qk_waits {:.0f}  qk_issue {:.0f}  P_wait {:.0f}  V_wait {:.0f}  "
          "pv_issue {:.0f}  loop {:.0f}".format(*d, np.diff(m[:, 0]).mean() - d.sum()))


if __name__ == "__main__":
    main()
