timeout 300 python scripts/classes.py 5 2>&1 | head -12
for w in "3 34" "4 34" "3 64" "6 34" "8 34" "4 128"; do set -- $w; echo "== workers $1 slice $2"; timeout 600 python bench.py --config 5 --steps 5 --no-cpu-baseline --workers $1 --slice $2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
