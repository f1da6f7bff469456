#!/bin/bash
# One gpurun call: build, GPU tests, bench, ncu launch list.  Usage (from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh TAG [tests|notests] [ncu|noncu]'
# Writes gpurun_out/TAG_{build,tests,bench,launches}.*
TAG=${1:-run}
TESTS=${2:-tests}
NCU=${3:-ncu}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/${TAG}_build.log; exit 1; }
if [ "$TESTS" = tests ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1
  echo "tests exit $?"; tail -5 gpurun_out/${TAG}_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1
  tail -2 gpurun_out/${TAG}_smoke.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?"; cat gpurun_out/${TAG}_bench.json; tail -5 gpurun_out/${TAG}_bench.err
if [ "$NCU" = ncu ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --dense-steps 1 \
    --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_bench.log 2>&1
  echo "ncu exit $?"
fi
