for keep in "" "130000000000"; do echo "== keep $keep"; GPS_POOL_KEEP_BYTES=$keep BENCH_DEBUG=1 timeout 600 python bench.py --config 3 --steps 12 --no-cpu-baseline 2>&1 | grep -E "^step" | tr '\n' ' '; echo; done
GPS_TRACE=1 timeout 600 python scripts/spikes.py 3 2> gpurun_out/spikes2.txt; grep STEP gpurun_out/spikes2.txt
