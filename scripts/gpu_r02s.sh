# r02s: cursor-batched tiled collect; ncu of the bulk join
mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q > gpurun_out/s_tests.log 2>&1; echo exit $? >> gpurun_out/s_tests.log)
tail -2 gpurun_out/s_tests.log
for i in 1 2; do
  echo "== cfg2"; timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'].get('kernel'), d['roofline']['achieved'], d['roofline']['frac'])"
done
timeout 300 python scripts/classes.py 2 2>&1 | head -10
CLASSES=1 timeout 600 python scripts/ncu_cfg4.py 2>&1 | tail -9
bash scripts/ncu_bulk.sh
