(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_budget.py -m gpu -x -q > gpurun_out/gpu_tests_j.log 2>&1; echo exit $? >> gpurun_out/gpu_tests_j.log)
tail -3 gpurun_out/gpu_tests_j.log
for w in 1 3; do echo "== workers $w"; BENCH_DEBUG=1 timeout 300 python bench.py --config 3 --steps 10 --workers $w --no-cpu-baseline 2>&1 | grep -E "^step" | tr '\n' ' '; echo; done
timeout 300 python scripts/classes.py 3 2>&1 | head -12
