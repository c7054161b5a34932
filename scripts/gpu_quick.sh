for d in 1 2 3 1; do echo "div $d"; GPS_GRID_DIV=$d python scripts/sweep_workers.py 2 | grep -v outlier | head -3; done
