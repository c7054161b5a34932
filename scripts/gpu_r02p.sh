# r02p: parity of the bulk-staged join write + one-block collect, then A/B bench lines.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash scripts/gpu_r02p.sh'
mkdir -p gpurun_out
(timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_budget.py \
    tests/test_gpu_commonsense.py tests/test_gpu_large.py -m gpu -x -q > gpurun_out/p_tests.log 2>&1; echo exit $? >> gpurun_out/p_tests.log)
tail -4 gpurun_out/p_tests.log
for e in "" "GPS_JOIN_NO_BULK=1" "GPS_COLLECT_TILED=1"; do
  echo "== cfg2 $e"; env $e timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'].get('kernel'), d['roofline']['achieved'], d['roofline']['frac'])"
done
for e in "" "GPS_JOIN_NO_BULK=1"; do
  echo "== cfg4 classes $e"; env $e CLASSES=1 timeout 600 python scripts/ncu_cfg4.py 2>&1 | tail -9
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:"k_join_bulk|k_join_seg" --csv python scripts/ncu_cfg4.py 2>/dev/null | grep -E "k_join" | \
  awk -F'","' '{print $5, $(NF-2), $(NF)}' | sed 's/"//g' | head -40
