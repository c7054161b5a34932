(timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q > gpurun_out/seg_tests.log 2>&1; echo exit $? >> gpurun_out/seg_tests.log)
tail -2 gpurun_out/seg_tests.log; grep -E "^E |FAILED" gpurun_out/seg_tests.log | head -5
timeout 300 python scripts/classes.py 2 2>&1 | grep -E "join_len|sum of"
CLASSES=1 timeout 600 python scripts/ncu_cfg4.py 2>&1 | tail -9 | grep -E "join_len"
timeout 300 python scripts/classes.py 5 2>&1 | grep -E "join_len"
for i in 1 2; do timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2', d['value'], r['kernel'], round(r['achieved']), round(r['frac'],4))"; done
timeout 600 python bench.py --config 5 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', d['value'])"
