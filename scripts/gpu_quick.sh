(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo exit $? >> gpurun_out/gpu_tests.log)
tail -2 gpurun_out/gpu_tests.log
python scripts/batch_classes.py 2 34 | head -10
CLASSES=1 python scripts/ncu_cfg4.py
timeout 400 python bench.py --config 5 --steps 5 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2> gpurun_out/bench_cfg5.err
tail -1 gpurun_out/bench_cfg5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['achieved'])"
