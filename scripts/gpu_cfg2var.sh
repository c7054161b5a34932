for r in "" 17179869184 "" 17179869184 "" 17179869184; do
  GPS_POOL_RESERVE_BYTES=$r BENCH_DEBUG=1 timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/tmp/err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('reserve=$r', d['value'], d['ms_per_step'])"
  grep "^step" /tmp/err.txt | awk '{print $3}' | sort -n | tail -3 | tr '\n' ' '; echo
done
