# One gpurun round trip: GPU parity tests, smoke, default bench line.
#   /usr/local/graft/bin/gpurun --timeout 1500 -- 'bash scripts/gpu_quick.sh'
(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo exit $? >> gpurun_out/gpu_tests.log)
tail -2 gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/bench_cfg2.log 2> gpurun_out/bench_cfg2.err
tail -1 gpurun_out/bench_cfg2.log | cut -c 1-300
