(timeout 900 python -m pytest tests/test_gpu_commonsense.py tests/test_gpu_parity.py tests/test_gpu_budget.py tests/test_gpu_large.py -m gpu -x -q > gpurun_out/gpu_tests_l.log 2>&1; echo exit $? >> gpurun_out/gpu_tests_l.log)
tail -3 gpurun_out/gpu_tests_l.log
CLASSES=1 timeout 600 python scripts/ncu_cfg4.py 2>&1 | tail -9
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_join_fast" --csv python scripts/ncu_cfg4.py 2>/dev/null | grep -E "k_join" | awk -F'","' '{print $5, $(NF-2), $(NF)}' | sed 's/"//g' | head -24
timeout 300 python scripts/classes.py 2 2>&1 | head -12
