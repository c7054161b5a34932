bash scripts/gpu_tests.sh
CLASSES=1 timeout 600 python scripts/ncu_cfg4.py 2>&1 | tail -9 | grep -E "join_len|join_write"
timeout 300 python scripts/classes.py 2 2>&1 | grep -E "join_len|sum of"
