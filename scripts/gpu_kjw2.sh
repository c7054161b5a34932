timeout 600 python scripts/classes.py 3 2>&1 | head -3 | tail -1
for i in 1 2; do timeout 600 python bench.py --config 3 --steps 6 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['value'], d['ms_per_step'])"; done
timeout 900 python bench.py --config 4 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', d['value'], d['ms_per_step'])"
timeout 600 python bench.py --config 5 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', d['value'], d['ms_per_step'])"
(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/kjw2_tests.log 2>&1; echo exit $? >> gpurun_out/kjw2_tests.log)
tail -2 gpurun_out/kjw2_tests.log
