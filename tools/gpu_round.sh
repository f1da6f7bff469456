#!/bin/bash
# One gpurun call: build, GPU tests + smoke, bench, ncu launch list, attention metrics,
# whole-call CPU oracle timings.  Usage (from the repo root):
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh TAG [tests|notests] [ncu|noncu] [cpu|nocpu]'
# Writes gpurun_out/TAG_*
TAG=${1:-run}
TESTS=${2:-tests}
NCU=${3:-ncu}
CPU=${4:-nocpu}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/${TAG}_build.log; exit 1; }
if [ "$TESTS" = tests ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1
  echo "tests exit $?"; tail -3 gpurun_out/${TAG}_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1
  tail -2 gpurun_out/${TAG}_smoke.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?"; cat gpurun_out/${TAG}_bench.json; tail -5 gpurun_out/${TAG}_bench.err
if [ "$NCU" = ncu ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --dense-steps 1 \
    --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_bench.log 2>&1
  echo "ncu launches exit $?"
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:sparse_attn_fwd -c 1 --csv --log-file gpurun_out/${TAG}_attn_metrics.csv \
    python bench.py --steps 1 --warmup 0 --dense-steps 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_attn.log 2>&1
  echo "ncu attention metrics exit $?"
fi
if [ "$CPU" = cpu ]; then
  timeout 900 python tools/cpu_oracle_bench.py --out gpurun_out/${TAG}_cpu_oracle.json > /dev/null 2> gpurun_out/${TAG}_cpu.err
  echo "cpu oracle exit $?"; cat gpurun_out/${TAG}_cpu_oracle.json
fi
