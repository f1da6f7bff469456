mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp13_launches.csv -k regex:"oz|split" python tools/score_bench.py > gpurun_out/exp13.log 2>&1
python tools/score_bench.py > gpurun_out/exp13_score.txt 2>&1; tail -1 gpurun_out/exp13_score.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -s -k "ozaki or scores or index_lists or topk_bit or end_to_end or waver_full" > gpurun_out/exp13_tests.txt 2>&1; grep -E "passed|failed|ozaki|Error" gpurun_out/exp13_tests.txt | head -40
