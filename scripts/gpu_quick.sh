nproc; python scripts/sweep_workers.py 2; python scripts/sweep_workers.py 2
