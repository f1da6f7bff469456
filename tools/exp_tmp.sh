mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tokens or tile_pool or host_pipeline" > gpurun_out/exp8_tests.txt 2>&1; tail -2 gpurun_out/exp8_tests.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/exp8_bench.json 2>&1; cat gpurun_out/exp8_bench.json
