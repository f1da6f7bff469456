#!/bin/bash
# Evidence for profiles/: ncu --set full of the path's kernels in bench.py's configuration,
# compute-sanitizer over small cases, and the sparsity sweep.  One gpurun call each:
#   gpurun --timeout 2400 -- 'bash tools/final_evidence.sh TAG ncu'
#   gpurun --timeout 2400 -- 'bash tools/final_evidence.sh TAG sanitize'
#   gpurun --timeout 3600 -- 'bash tools/final_evidence.sh TAG sweep'
# Writes gpurun_out/TAG_*
TAG=${1:-final}
WHAT=${2:-ncu}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/${TAG}_build.log; exit 1; }
B="python bench.py --steps 1 --warmup 1 --dense-steps 1 --no-cpu-baseline --no-e2e"
case "$WHAT" in
ncu)
  # attention: one launch of the token-layout kernel at Waver / 24 heads (the bench's)
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:sparse_attn_fwd -s 1 -c 1 \
    -o gpurun_out/${TAG}_attn_full -f $B > gpurun_out/${TAG}_attn_full.log 2>&1
  echo "attn full exit $?"
  # the other steps: pool, Ozaki GEMMs / splits, top-k (second call of the step, warm)
  timeout 900 ncu --set full --clock-control none -k regex:'pool_tma|oz_gemm|split_rows|split_cols|topk_filter' \
    -s 11 -c 11 -o gpurun_out/${TAG}_steps_full -f $B > gpurun_out/${TAG}_steps_full.log 2>&1
  echo "steps full exit $?"
  for r in attn_full steps_full; do
    python tools/ncu_summary.py gpurun_out/${TAG}_${r}.ncu-rep sm__pipe_tensor smsp__pcsamp > gpurun_out/${TAG}_${r}.txt 2>&1
  done
  ;;
sanitize)
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool python tools/sanitize_path.py > gpurun_out/${TAG}_san_${tool}.txt 2>&1
    echo "$tool exit $?"; tail -3 gpurun_out/${TAG}_san_${tool}.txt
  done
  ;;
sweep)
  timeout 3300 python tools/sweep.py --shards --out gpurun_out/${TAG}_sweep > gpurun_out/${TAG}_sweep.log 2>&1
  echo "sweep exit $?"; tail -25 gpurun_out/${TAG}_sweep.md
  ;;
esac
