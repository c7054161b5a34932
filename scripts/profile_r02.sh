#!/bin/bash
# Round-2 evidence: launch list of the default bench (cfg2), full captures of the cfg2 batch kernels,
# of the cfg3 join kernels and of the cfg4 joins; summaries into gpurun_out/profiles/.
R=${1:-r02}
mkdir -p gpurun_out/profiles
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_$R.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/profiles/${R}_bench_under_ncu.log 2>&1
MODE=match SLICE=34 timeout 1200 ncu -f --set full --import-source on --clock-control none \
    -k regex:"k_check|k_collect|k_explore|k_post|k_ec|k_join" -c 60 -o /tmp/prof_${R}_cfg2 python scripts/ncu_target.py \
    > gpurun_out/profiles/${R}_ncu_cfg2.log 2>&1
PASSES=1 timeout 1200 ncu -f --set full --import-source on --clock-control none -k regex:"k_join_v|k_join<|k_join_seg|k_ec|k_explore" \
    -c 40 -o /tmp/prof_${R}_cfg3 python scripts/ncu_cfg3.py > gpurun_out/profiles/${R}_ncu_cfg3.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_join|k_ec|k_explore|k_check|k_collect" -c 24 \
    -o /tmp/prof_${R}_cfg4 python scripts/ncu_cfg4.py > gpurun_out/profiles/${R}_ncu_cfg4.log 2>&1
TRAFFIC_PREFIX=cfg2: python scripts/summarize_profiles.py ${R}_cfg2 /tmp/launches_$R.csv /tmp/prof_${R}_cfg2.ncu-rep > /dev/null
TRAFFIC_PREFIX=cfg3: python scripts/summarize_profiles.py ${R}_cfg3 /tmp/launches_$R.csv /tmp/prof_${R}_cfg3.ncu-rep > /dev/null
TRAFFIC_PREFIX=cfg4: python scripts/summarize_profiles.py ${R}_cfg4 /tmp/launches_$R.csv /tmp/prof_${R}_cfg4.ncu-rep > /dev/null
cp profiles/${R}_* profiles/traffic.json gpurun_out/profiles/
ls -la gpurun_out/profiles; du -sh gpurun_out
