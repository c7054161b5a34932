#!/bin/bash
# Bench lines of every config (+ the reference arm) into gpurun_out/profiles/<R>_bench_*.json.
R=${1:-r02b}
mkdir -p gpurun_out/profiles
timeout 600 python bench.py > gpurun_out/profiles/${R}_bench_cfg2.json 2> gpurun_out/profiles/${R}_bench_cfg2.err
tail -1 gpurun_out/profiles/${R}_bench_cfg2.json | cut -c 1-200
timeout 900 python bench.py --config 3 --steps 10 > gpurun_out/profiles/${R}_bench_cfg3.json 2> gpurun_out/profiles/${R}_bench_cfg3.err
tail -1 gpurun_out/profiles/${R}_bench_cfg3.json | cut -c 1-200
timeout 1200 python bench.py --config 4 --steps 5 > gpurun_out/profiles/${R}_bench_cfg4.json 2> gpurun_out/profiles/${R}_bench_cfg4.err
tail -1 gpurun_out/profiles/${R}_bench_cfg4.json | cut -c 1-200
timeout 900 python bench.py --config 5 --steps 5 > gpurun_out/profiles/${R}_bench_cfg5.json 2> gpurun_out/profiles/${R}_bench_cfg5.err
tail -1 gpurun_out/profiles/${R}_bench_cfg5.json | cut -c 1-200
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/profiles/${R}_bench_reference.json 2>&1
tail -1 gpurun_out/profiles/${R}_bench_reference.json | cut -c 1-200
