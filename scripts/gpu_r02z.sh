mkdir -p gpurun_out
(timeout 1500 python -m pytest tests/test_gpu_relate.py tests/test_gpu_parity.py tests/test_gpu_budget.py tests/test_gpu_configs.py tests/test_gpu_large.py -m gpu -x -q > gpurun_out/z_tests.log 2>&1; echo exit $? >> gpurun_out/z_tests.log)
tail -3 gpurun_out/z_tests.log; grep -E "^E |FAILED" gpurun_out/z_tests.log | head -10
timeout 600 python scripts/cfg4_steps.py batch 2>/dev/null | tail -6
for i in 1 2; do BENCH_DEBUG=1 timeout 900 python bench.py --config 4 --steps 5 --no-cpu-baseline 2>&1 | grep -E "^step|queries/s" | cut -c 1-120 | tail -6; done
