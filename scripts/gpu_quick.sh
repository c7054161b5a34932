timeout 400 python bench.py > gpurun_out/bench_cfg2.log 2> gpurun_out/bench_cfg2.err
timeout 400 python bench.py --config 5 --steps 5 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2> gpurun_out/bench_cfg5.err
timeout 400 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2> gpurun_out/bench_cfg3.err
timeout 400 python bench.py > gpurun_out/bench_cfg2b.log 2> gpurun_out/bench_cfg2b.err
for c in 2 3 5 2b; do tail -1 gpurun_out/bench_cfg$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), round(d['ms_per_step'],3), '%.3g'%d['embeddings_per_s'], d['roofline']['kernel'], round(d['roofline']['achieved'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1), d.get('cpu_baseline',{}).get('value'), d['clocks']['reasons'], d.get('latency_ms',{}).get('p99'))"; done
