# Full ncu capture of the cfg4 bulk join write (the two largest launches) + cfg2 collect, read back here.
mkdir -p gpurun_out
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_join_bulk<3>" -c 2 \
    -o gpurun_out/prof_bulk3 python scripts/ncu_cfg4.py > gpurun_out/ncu_bulk.log 2>&1; echo "ncu rc $?"
MODE=match SLICE=34 timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_collect|k_join_bulk" -c 12 \
    -o gpurun_out/prof_cfg2 python scripts/ncu_target.py > gpurun_out/ncu_cfg2.log 2>&1; echo "ncu rc $?"
ls -la gpurun_out/*.ncu-rep
