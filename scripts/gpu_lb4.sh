(timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus or cfg2" > gpurun_out/lb4_tests.log 2>&1; echo exit $? >> gpurun_out/lb4_tests.log)
tail -2 gpurun_out/lb4_tests.log
timeout 300 python scripts/classes.py 2 2>&1 | grep join_write
CLASSES=1 timeout 600 python scripts/ncu_cfg4.py 2>&1 | tail -9 | head -1
for i in 1 2; do timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])"; done
timeout 900 python bench.py --config 4 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', d['value'], d['ms_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_join_bulk" --csv python scripts/ncu_cfg4.py 2>/dev/null | grep -E "k_join" | awk -F'","' '{print $5, $(NF-2), $(NF)}' | sed 's/"//g' | grep -E "pct|duration" | head -8
