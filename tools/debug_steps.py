"""Step-by-step smoke of every libveda kernel with a sync and a flush after each one
(first thing to run on a new GPU box; isolates hangs and faults).

    python tools/debug_steps.py [case]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2605_30325_b200 import build, synth, veda  # noqa: E402

CASES = {
    "tiny": ((4, 8, 8), [(4, 4, 4)], 64, 1, 2),
    "b128": ((5, 9, 14), [(4, 4, 8)], 128, 2, 4),
    "b64d128": ((3, 5, 6), [(4, 4, 4)], 128, 2, 2),
    "b128d64": ((8, 12, 20), [(4, 4, 8)], 64, 3, 5),
}


def log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


def u16(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def main(name):
    lat, cfgs, d, Hh, kk = CASES[name]
    build.build()
    veda.load()
    veda.check_device()
    dev = torch.device("cuda")
    pre = synth.Preset(name, lat, Hh, d, cfgs[0], 0.5)
    q, k, v = synth.qkv(pre, lat=lat, d=d)
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre, d=d).items()}
    qd, kd, vd = q.to(dev), k.to(dev), v.to(dev)
    qt, cnt, mask = veda.tile_permute(qd, lat, cfgs)
    kt, _, _ = veda.tile_permute(kd, lat, cfgs, meta=False)
    vt, _, _ = veda.tile_permute(vd, lat, cfgs, meta=False)
    torch.cuda.synchronize()
    oq, ocnt, omask = oracle.tile_permute(u16(q), lat, cfgs)
    log(f"permute ok, bit-exact={np.array_equal(u16(qt), oq)} cnt={cnt.flatten()[:8].tolist()}")
    s = veda.tile_score(qt, kt, cnt, mask, veda.make_scorer(w))
    torch.cuda.synchronize()
    log(f"score ok, S[0,0,:4]={s[0, 0, :4].tolist()}")
    idx = veda.select_topk(s, kk)
    torch.cuda.synchronize()
    log(f"topk ok, idx[0,:2]={idx[0, :2].tolist()}")
    NT = qt.shape[1]
    for label, ii in (("sparse", idx), ("dense", torch.arange(NT, dtype=torch.int32, device=dev).expand(Hh, NT, NT).contiguous())):
        o = veda.sparse_attn_fwd(qt, kt, vt, ii, mask)
        torch.cuda.synchronize()
        ref = oracle.sparse_attn(oq, oracle.tile_permute(u16(k), lat, cfgs)[0], oracle.tile_permute(u16(v), lat, cfgs)[0],
                                 ii.cpu().numpy(), omask)
        og = oracle.bf16_bits_to_f64(u16(o))
        B = qt.shape[2]
        real = ((omask[..., :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(Hh, NT, -1)[..., :B].astype(bool)
        err = np.abs(og[real] - ref[real])
        log(f"attn {label} ok: max err {err.max():.3e} mean {err.mean():.3e}; o[0,0,0,:4]={og[0,0,0,:4]} ref={ref[0,0,0,:4]}")
    ot = veda.tile_unpermute(o, lat, cfgs)
    torch.cuda.synchronize()
    log("unpermute ok")


if __name__ == "__main__":
    for n in (sys.argv[1:] or list(CASES)):
        log(f"=== {n}")
        main(n)
