"""Write profiles/attn_traffic.json (DRAM bytes per launch of the path's attention kernel,
read by bench.py's roofline.traffic) and print the raw tensor-pipe / DRAM metrics, from an
ncu CSV of the attention launch in bench.py's configuration:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,\\
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,\\
sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,\\
sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct \\
        --clock-control none -k regex:sparse_attn_fwd -c 1 --csv --log-file gpurun_out/attn_metrics.csv \\
        python bench.py --steps 1 --warmup 0 --dense-steps 1 --no-cpu-baseline --no-e2e
    python tools/ncu_attn_traffic.py gpurun_out/attn_metrics.csv [--heads 24] [--workload waver12b]
"""
import argparse
import csv
import json
import os


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--heads", type=int, default=24)
    ap.add_argument("--workload", default="waver12b")
    ap.add_argument("--tree", default="")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
    h = rows[0]
    vals = {}
    for r in rows[1:]:
        if "sparse_attn_fwd" not in r[h.index("Kernel Name")]:
            continue
        try:
            vals[r[h.index("Metric Name")]] = (float(r[h.index("Metric Value")].replace(",", "")),
                                               r[h.index("Metric Unit")])
        except ValueError:
            pass
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = vals["dram__bytes_read.sum"]
    wr = vals["dram__bytes_write.sum"]
    dram = rd[0] * scale[rd[1]] + wr[0] * scale[wr[1]]
    out = {"workload": a.workload, "heads_per_launch": a.heads, "dram_bytes_per_launch": dram,
           "source": "ncu dram__bytes_read.sum + dram__bytes_write.sum, one launch of the bench's attention",
           "tree": a.tree, "metrics": {k: v[0] for k, v in vals.items()}}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "profiles", "attn_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
