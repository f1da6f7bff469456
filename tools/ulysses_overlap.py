"""Ulysses front end (ulysses.py) on one GPU through NCCL (world size 1): per-call time for
several chunk counts against the direct call, and the event timeline of one chunked call on
the compute stream (when each chunk's inputs were usable vs when the previous chunk's path
finished: with the exchange overlapped, chunk c+1's inputs are in before chunk c's path ends).

    python tools/ulysses_overlap.py [--workload waver12b] [--chunks 1 3 6 12]
"""
import argparse
import json
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import synth, ulysses, veda  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="waver12b")
    ap.add_argument("--chunks", type=int, nargs="+", default=[1, 3, 6, 12])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    veda.load()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
    s.close()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    pre = synth.PRESETS[a.workload]
    w = {n: t.to(dev) for n, t in synth.scorer_weights(pre).items()}
    q, k, v = synth.qkv(pre, device=dev, layout="nhd")  # [N, Hh, d]: the sequence-shard layout

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    direct = veda.SparseAttention(pre.lat, [pre.cfg], pre.heads, pre.d, w, sparsity=pre.sparsity, device=dev)
    out = torch.empty_like(q)
    res = {"workload": a.workload, "world": 1,
           "direct_ms": round(timed(lambda: direct(q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1),
                                                   out=out.transpose(0, 1))), 3)}
    del direct
    torch.cuda.empty_cache()
    for C in a.chunks:
        up = ulysses.UlyssesSparseAttention(pre.lat, [pre.cfg], pre.heads, pre.d, w, sparsity=pre.sparsity,
                                            device=dev, chunks=C)
        res[f"ulysses_chunks{C}_ms"] = round(timed(lambda: up(q, k, v)), 3)
        if C == max(a.chunks):
            tr = []
            up(q, k, v, trace=tr)
            torch.cuda.synchronize()
            t0 = tr[0][1]
            res[f"timeline_chunks{C}_ms"] = [(lab, round(t0.elapsed_time(e), 3)) for lab, e in tr]
        del up
        torch.cuda.empty_cache()
    dist.destroy_process_group()
    line = json.dumps(res, indent=1)
    print(line)
    if a.out:
        open(a.out, "w").write(line + "\n")


if __name__ == "__main__":
    main()
