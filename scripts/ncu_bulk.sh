# Full ncu captures of the bulk join write: cfg4 (the first four launches: two large <3> writes)
# and one cfg2 batch.  Reports land in gpurun_out/ and are read back here.
mkdir -p gpurun_out
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_join_bulk" -c 4 \
    -o gpurun_out/prof_bulk_cfg4 python scripts/ncu_cfg4.py > gpurun_out/ncu_bulk.log 2>&1; echo "ncu rc $?"
MODE=match SLICE=34 timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_join_bulk" -c 10 \
    -o gpurun_out/prof_bulk_cfg2 python scripts/ncu_target.py > gpurun_out/ncu_cfg2.log 2>&1; echo "ncu rc $?"
ls -la gpurun_out/*.ncu-rep
