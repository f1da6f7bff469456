"""Whole-call timings of the fp64 CPU oracle: every head and every
query tile of the tiny, Wan2.1-1.3B and (--wan14b) Wan2.1-14B workloads on this host's cores, plus a single-thread
figure, next to the bounded Waver sample that bench.py's cpu_baseline uses.  A reported
baseline, not a target.

    python tools/cpu_oracle_bench.py [--out profiles/r02_cpu_oracle.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--skip-wan", action="store_true")
    ap.add_argument("--wan14b", action="store_true", help="also the whole Wan2.1-14B call (~3 min on 16 cores)")
    a = ap.parse_args()
    from paper_2605_30325_b200 import synth

    cores = len(os.sched_getaffinity(0))
    res = {"cpu_model": bench.cpu_model(), "cores": cores, "kind": "oracle (fp64 C, plain loops, pthreads over "
           "query tiles)", "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    res["tiny_full_call_ms"] = round(bench.oracle_full("tiny"), 2)
    if not a.skip_wan:
        res["wan1.3b_full_call_ms"] = round(bench.oracle_full("wan1.3b"), 1)
    if a.wan14b:
        res["wan14b_full_call_ms"] = round(bench.oracle_full("wan14b"), 1)
    pre = synth.PRESETS["waver12b"]
    ms, cores, sample, wall, single = bench.oracle_sample(pre, pre.sparsity, 240, single_thread_units=8)
    res["waver12b_extrapolated_ms"] = round(ms, 1)
    res["waver12b_single_thread_extrapolated_ms"] = round(single, 1)
    res["waver12b_sample"] = sample
    line = json.dumps(res, indent=1)
    print(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
