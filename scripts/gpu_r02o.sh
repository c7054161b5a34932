mkdir -p gpurun_out/profiles
timeout 600 compute-sanitizer --tool initcheck --print-limit 50 --error-exitcode 9 python scripts/sanitize_target.py > gpurun_out/profiles/r02_sanitizer_initcheck_after_fix.txt 2>&1; echo "initcheck exit $?"
tail -2 gpurun_out/profiles/r02_sanitizer_initcheck_after_fix.txt
for e in "" "GPS_NO_CLOSE_DIR=1"; do echo "== cfg5 $e"; env $e timeout 600 python bench.py --config 5 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c 100-200; done
for e in "" "GPS_NO_CLOSE_DIR=1"; do echo "== cfg2 $e"; env $e timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c 100-200; done
for e in "GPS_JOIN_ORDER=paper" "GPS_JOIN_ORDER=constrained"; do echo "== cfg3 $e"; env $e timeout 300 python scripts/trace_cfg.py 3 1 34 2>&1 | grep -E "step wall|pairs" | head -14; done
GPS_JOIN_ORDER=constrained timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "cfg3_cyclic_counts" 2>&1 | tail -1
GPS_JOIN_ORDER=constrained BENCH_DEBUG=1 timeout 600 python bench.py --config 3 --steps 6 --no-cpu-baseline 2>&1 | grep -E "^step" | tr '\n' ' '
