(timeout 600 python -m pytest tests/test_gpu_commonsense.py -m gpu -x -q > gpurun_out/gpu_tests_m.log 2>&1; echo exit $? >> gpurun_out/gpu_tests_m.log)
tail -2 gpurun_out/gpu_tests_m.log
bash scripts/sanitize.sh
