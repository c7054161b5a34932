(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo exit $? >> gpurun_out/gpu_tests.log)
tail -4 gpurun_out/gpu_tests.log
timeout 300 python scripts/classes.py 2 > gpurun_out/classes_cfg2.txt 2>&1
timeout 600 python scripts/classes.py 3 > gpurun_out/classes_cfg3.txt 2>&1
cat gpurun_out/classes_cfg3.txt | head -20
timeout 400 python bench.py --steps 20 > gpurun_out/bench_cfg2.log 2> gpurun_out/bench_cfg2.err
tail -1 gpurun_out/bench_cfg2.log | cut -c 1-300
timeout 900 python bench.py --config 3 --steps 5 > gpurun_out/bench_cfg3.log 2> gpurun_out/bench_cfg3.err
tail -1 gpurun_out/bench_cfg3.log | cut -c 1-300
