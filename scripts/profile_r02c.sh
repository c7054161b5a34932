#!/bin/bash
# Round evidence r02c: launch list of the default bench (cfg2), full captures of one cfg2 batch
# slice and of the cfg4 kernels, summarised into profiles/ and copied back via gpurun_out/.
R=${1:-r02c}
mkdir -p gpurun_out/profiles
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_$R.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/profiles/${R}_bench_under_ncu.log 2>&1
echo "launch list rc $?"
MODE=match SLICE=34 timeout 1200 ncu -f --set full --import-source on --clock-control none \
    -k regex:"k_check|k_collect|k_explore|k_ec|k_join" -c 60 -o /tmp/prof_${R}_cfg2 python scripts/ncu_target.py \
    > gpurun_out/profiles/${R}_ncu_cfg2.log 2>&1
echo "cfg2 capture rc $?"
timeout 1500 ncu -f --set full --import-source on --clock-control none \
    -k regex:"k_check|k_collect|k_explore|k_ec|k_join" -c 40 -o /tmp/prof_${R}_cfg4 python scripts/ncu_cfg4.py \
    > gpurun_out/profiles/${R}_ncu_cfg4.log 2>&1
echo "cfg4 capture rc $?"
PASSES=1 timeout 1200 ncu -f --set full --import-source on --clock-control none \
    -k regex:"k_join|k_explore|k_collect|k_ec" -c 40 -o /tmp/prof_${R}_cfg3 python scripts/ncu_cfg3.py \
    > gpurun_out/profiles/${R}_ncu_cfg3.log 2>&1
echo "cfg3 capture rc $?"
TRAFFIC_PREFIX=cfg3: python scripts/summarize_profiles.py ${R}_cfg3 /tmp/launches_$R.csv /tmp/prof_${R}_cfg3.ncu-rep > /dev/null
TRAFFIC_PREFIX=cfg2: python scripts/summarize_profiles.py ${R}_cfg2 /tmp/launches_$R.csv /tmp/prof_${R}_cfg2.ncu-rep > /dev/null
TRAFFIC_PREFIX=cfg4: python scripts/summarize_profiles.py ${R}_cfg4 /tmp/launches_$R.csv /tmp/prof_${R}_cfg4.ncu-rep > /dev/null
cp profiles/${R}_* profiles/traffic.json gpurun_out/profiles/
ls -la /tmp/prof_${R}_cfg4.ncu-rep /tmp/prof_${R}_cfg2.ncu-rep
ls -la gpurun_out/profiles | tail; du -sh gpurun_out
