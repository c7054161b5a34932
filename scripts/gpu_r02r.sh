# r02r: batched-gather smem collect A/B
mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus or cfg2" > gpurun_out/r_tests.log 2>&1; echo exit $? >> gpurun_out/r_tests.log)
tail -2 gpurun_out/r_tests.log
for e in "" "GPS_COLLECT_TILED=1" "" "GPS_COLLECT_TILED=1"; do
  echo "== cfg2 $e"; env $e timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'].get('kernel'), d['roofline']['achieved'], d['roofline']['frac'])"
done
for e in "" "GPS_COLLECT_TILED=1"; do echo "== classes $e"; env $e timeout 300 python scripts/classes.py 2 2>&1 | head -10; done
