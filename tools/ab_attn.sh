#!/bin/bash
# usage: bash ab.sh TAG "testexpr" lib1 lib2 ...
TAG=$1; shift; TEXPR=$1; shift
mkdir -p gpurun_out
if [ -n "$TEXPR" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$TEXPR" > gpurun_out/${TAG}_tests.log 2>&1
  echo "tests exit $?"; tail -3 gpurun_out/${TAG}_tests.log
fi
for rep in 1 2 3; do
  for lib in "$@"; do
    VEDA_LIB=$PWD/paper_2605_30325_b200/$lib timeout 300 python tools/attn_bench.py --heads 24 --tokens --reps 5 2>&1 | tail -1
  done
done
for lib in $TRACE_LIBS; do
  echo "== trace $lib"
  VEDA_LIB=$PWD/paper_2605_30325_b200/$lib timeout 300 python tools/attn_trace.py --heads 4 2>&1 | tail -40
done
