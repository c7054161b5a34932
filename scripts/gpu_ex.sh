(timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus or cfg2 or filter" > gpurun_out/ex_tests.log 2>&1; echo exit $? >> gpurun_out/ex_tests.log)
tail -2 gpurun_out/ex_tests.log
timeout 300 python scripts/classes.py 2 2>&1 | grep -E "explore|propagate|collect|sum of"
CLASSES=1 timeout 600 python scripts/ncu_cfg4.py 2>&1 | tail -9 | grep -E "explore|propagate|collect"
for i in 1 2; do timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2', d['value'], r['kernel'], round(r['achieved']), round(r['frac'],4))"; done
