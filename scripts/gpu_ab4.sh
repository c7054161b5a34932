for d in . alt11 . alt11; do
  echo "== $d"; (cd $d && BENCH_DEBUG=1 timeout 900 python bench.py --config 4 --steps 5 --no-cpu-baseline 2>&1 | grep -E "^step|queries/s" | cut -c 1-160 | tail -8)
done
