(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/wide_tests.log 2>&1; echo exit $? >> gpurun_out/wide_tests.log)
tail -2 gpurun_out/wide_tests.log; grep -E "^E |FAILED" gpurun_out/wide_tests.log | head
for e in "" "GPS_JOIN_WIDE_STAGED=0" "" "GPS_JOIN_WIDE_STAGED=0"; do
  echo "== $e"; env $e timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'].get('kernel'), d['roofline']['achieved'], d['roofline']['frac'])"
  env $e timeout 300 python scripts/classes.py 2 2>&1 | grep join_write
done
for e in "" "GPS_JOIN_WIDE_STAGED=0"; do echo "== cfg5 $e"; env $e timeout 600 python bench.py --config 5 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
