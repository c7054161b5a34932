(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/kjw_tests.log 2>&1; echo exit $? >> gpurun_out/kjw_tests.log)
tail -2 gpurun_out/kjw_tests.log; grep -E "^E |FAILED" gpurun_out/kjw_tests.log | head
timeout 600 python scripts/classes.py 3 2>&1 | head -4
for i in 1 2; do timeout 600 python bench.py --config 3 --steps 6 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', d['value'], d['ms_per_step'])"
timeout 900 python bench.py --config 4 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', d['value'], d['ms_per_step'])"
