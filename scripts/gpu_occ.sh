(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/occ_tests.log 2>&1; echo exit $? >> gpurun_out/occ_tests.log)
tail -2 gpurun_out/occ_tests.log; grep -E "^E |FAILED" gpurun_out/occ_tests.log | head -5
timeout 300 python scripts/classes.py 2 2>&1 | head -10
CLASSES=1 timeout 600 python scripts/ncu_cfg4.py 2>&1 | tail -9 | head -7
for i in 1 2; do timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'])"; done
timeout 600 python bench.py --config 5 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', d['value'], d['ms_per_step'])"
timeout 900 python bench.py --config 4 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', d['value'], d['ms_per_step'])"
timeout 600 python bench.py --config 3 --steps 6 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['value'], d['ms_per_step'])"
