#!/bin/bash
# Round evidence: launch list of the default bench, full captures of one cfg2 batch (bench slicing)
# and of the cfg4 joins, summarised into profiles/ and copied to gpurun_out/ (profiles/ on the box
# does not travel back).   usage: bash scripts/profile_round.sh ROUND
R=${1:-r01d}
mkdir -p gpurun_out/profiles
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_$R.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/profiles/${R}_bench_under_ncu.log 2>&1
MODE=match SLICE=34 timeout 1200 ncu -f --set full --import-source on --clock-control none \
    -k regex:"k_check|k_collect|k_explore|k_post|k_ec|k_join" -o /tmp/prof_${R}_cfg2 python scripts/ncu_target.py \
    > gpurun_out/profiles/${R}_ncu_cfg2.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_join" -c 12 \
    -o /tmp/prof_${R}_cfg4 python scripts/ncu_cfg4.py > gpurun_out/profiles/${R}_ncu_cfg4.log 2>&1
python scripts/summarize_profiles.py $R /tmp/launches_$R.csv /tmp/prof_${R}_cfg2.ncu-rep > /dev/null
TRAFFIC_PREFIX=cfg4: python scripts/summarize_profiles.py ${R}_cfg4 /tmp/launches_$R.csv /tmp/prof_${R}_cfg4.ncu-rep > /dev/null
cp profiles/${R}_* profiles/traffic.json gpurun_out/profiles/
python scripts/ncu_lines.py /tmp/prof_${R}_cfg4.ncu-rep gpurun_out/profiles/${R}_cfg4_lines 12 > /dev/null 2>&1
ls -la gpurun_out/profiles; du -sh gpurun_out
