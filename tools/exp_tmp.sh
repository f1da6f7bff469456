mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --clock-control none -k regex:"oz|split" --metrics gpu__time_duration.sum --csv --log-file gpurun_out/exp19.csv python tools/score_bench.py > gpurun_out/exp18.log 2>&1
echo rc $?
