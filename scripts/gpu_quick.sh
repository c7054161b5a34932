timeout 400 python bench.py > gpurun_out/bench_cfg2.log 2> gpurun_out/bench_cfg2.err
timeout 400 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2> gpurun_out/bench_cfg3.err
timeout 400 python bench.py --config 5 --steps 5 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --config 4 --steps 5 > gpurun_out/bench_cfg4.log 2> gpurun_out/bench_cfg4.err
for c in 2 3 5 4; do tail -1 gpurun_out/bench_cfg$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, round(d['value'],1), round(d['ms_per_step'],3), d['embeddings_per_s'], d['roofline']['kernel'], round(d['roofline']['achieved'],1), d['roofline']['traffic'], d['e2e']['value'], d.get('cpu_baseline',{}).get('value'))"; done
bash scripts/profile_round.sh r01b
