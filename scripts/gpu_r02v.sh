mkdir -p gpurun_out
(timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/v_tests.log 2>&1; echo exit $? >> gpurun_out/v_tests.log)
tail -2 gpurun_out/v_tests.log; grep -E "^E |FAILED|Error" gpurun_out/v_tests.log | head -10
for i in 1 2; do
  echo "== cfg2"; timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'].get('kernel'), d['roofline']['achieved'], d['roofline']['frac'])"
done
CLASSES=1 timeout 600 python scripts/ncu_cfg4.py 2>&1 | tail -9 | head -2
echo "== cfg4 bench"; timeout 900 python bench.py --config 4 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'].get('kernel'), d['roofline']['achieved'], d['roofline']['frac'])"
