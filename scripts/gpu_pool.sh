for r in "" 100000000000; do
  echo "== reserve '$r'"
  GPS_POOL_RESERVE_BYTES=$r timeout 600 python scripts/cfg4_steps.py batch 2>/dev/null | tail -12 | cut -c 1-40 | tr '\n' ' '; echo
  GPS_POOL_RESERVE_BYTES=$r BENCH_DEBUG=1 timeout 900 python bench.py --config 3 --steps 10 --no-cpu-baseline 2>&1 | grep -E "^step|queries/s" | cut -c 1-100 | tr '\n' ' '; echo
done
bash scripts/sanitize.sh r02c
