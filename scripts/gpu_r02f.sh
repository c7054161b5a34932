mkdir -p gpurun_out
(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1; echo exit $? >> gpurun_out/f_tests.log)
tail -3 gpurun_out/f_tests.log; grep -E "^E |FAILED" gpurun_out/f_tests.log | head -10
timeout 300 python scripts/classes.py 2 2>&1 | head -10
CLASSES=1 timeout 600 python scripts/ncu_cfg4.py 2>&1 | tail -9 | head -3
for i in 1 2; do timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'].get('kernel'), d['roofline']['achieved'], d['roofline']['frac'])"; done
timeout 900 python bench.py --config 4 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'].get('kernel'), d['roofline']['achieved'], d['roofline']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_join_bulk" --csv python scripts/ncu_cfg4.py 2>/dev/null | grep -E "k_join" | awk -F'","' '{print $5, $(NF-2), $(NF)}' | sed 's/"//g' | grep -E "pct|duration" | head -8
