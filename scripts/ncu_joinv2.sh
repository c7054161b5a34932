mkdir -p gpurun_out
PASSES=1 timeout 1200 ncu -f --set full --import-source on --clock-control none -k regex:"k_join" --launch-skip 17 --launch-count 1 -o gpurun_out/prof_join2 python scripts/ncu_cfg3.py > gpurun_out/ncu_join2.log 2>&1; echo rc $?
ls -la gpurun_out/prof_join2.ncu-rep
