timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k recovers 2>&1 | tail -15
timeout 300 python scripts/repro_big.py 11 0,1 2>&1 | tail -3
