mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus or cfg2" > gpurun_out/t_tests.log 2>&1; echo exit $? >> gpurun_out/t_tests.log)
tail -2 gpurun_out/t_tests.log
for i in 1 2; do
  echo "== cfg2"; timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'].get('kernel'), d['roofline']['achieved'], d['roofline']['frac'])"
done
timeout 300 python scripts/classes.py 2 2>&1 | head -10
bash scripts/ncu_bulk.sh
