(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_budget.py tests/test_gpu_sharded.py -m gpu -x -q > gpurun_out/gpu_tests_h.log 2>&1; echo exit $? >> gpurun_out/gpu_tests_h.log)
tail -3 gpurun_out/gpu_tests_h.log
timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k cfg3 2>&1 | tail -2
for spb in 0 4e9; do echo "== single-pass bytes $spb (0 = default)"; if [ "$spb" = "0" ]; then unset GPS_SINGLE_PASS_BYTES; else export GPS_SINGLE_PASS_BYTES=$spb; fi
  BENCH_DEBUG=1 timeout 300 python bench.py --config 3 --steps 10 --workers 3 --no-cpu-baseline 2>&1 | grep -E "^step" | tr '\n' ' '; echo; done
unset GPS_SINGLE_PASS_BYTES
timeout 300 python scripts/trace_cfg.py 3 1 34 2>&1 | grep -E "step wall|pairs" | head -14
