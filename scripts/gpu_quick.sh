(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo exit $? >> gpurun_out/gpu_tests.log)
tail -2 gpurun_out/gpu_tests.log
python scripts/batch_classes.py 2 34 > gpurun_out/classes_cfg2.txt 2>&1; head -11 gpurun_out/classes_cfg2.txt
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.log 2> gpurun_out/bench_cfg2.err
tail -1 gpurun_out/bench_cfg2.log | cut -c 1-250
