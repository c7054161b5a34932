# Round-2 baseline round trip: GPU tests, smoke, cfg2 + cfg4 bench lines, launch list of the default bench.
(timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo exit $? >> gpurun_out/gpu_tests.log)
tail -2 gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/bench_cfg2.log 2> gpurun_out/bench_cfg2.err
tail -1 gpurun_out/bench_cfg2.log | cut -c 1-400
timeout 600 python bench.py --config 4 --steps 5 > gpurun_out/bench_cfg4.log 2> gpurun_out/bench_cfg4.err
tail -1 gpurun_out/bench_cfg4.log | cut -c 1-400
nproc; lscpu | head -20 > gpurun_out/lscpu.txt
