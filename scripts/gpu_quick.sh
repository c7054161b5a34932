(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo exit $? >> gpurun_out/gpu_tests.log)
tail -2 gpurun_out/gpu_tests.log
timeout 300 python scripts/cfg5_warm.py
timeout 300 python scripts/cfg5_warm.py
python scripts/sweep_workers.py 2 | grep -v outlier | head -3
