for i in 1 2; do
(cd _wt/prev && python scripts/sweep_workers.py 2 | grep "workers=3" | sed 's/^/prev /')
python scripts/sweep_workers.py 2 | grep "workers=3" | sed 's/^/cur  /'
done
