"""Time veda_tile_pool (TripPool straight from token order) alone on a paper workload.

    python tools/pool_bench.py [--workload waver12b] [--heads 24] [--reps 20]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_30325_b200 import synth, veda  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="waver12b")
    ap.add_argument("--heads", type=int, default=24)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--layout", default="hnd")
    a = ap.parse_args()
    veda.load()
    pre = synth.PRESETS[a.workload]
    dev = torch.device("cuda")
    q, _, _ = synth.qkv(pre, heads=list(range(a.heads)), device=dev, layout=a.layout)
    if a.layout == "nhd":
        q = q.transpose(0, 1)
    z, cnt, mask = veda.tile_pool(q, pre.lat, [pre.cfg])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        veda.tile_pool(q, pre.lat, [pre.cfg], z=z)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    nbytes = q.numel() * 2 + z.numel() * 4
    print(f"tile_pool {a.workload} heads={a.heads} {a.layout}: {ms * 1e3:.1f} us, {nbytes / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
