python scripts/batch_classes.py 2 25 > gpurun_out/classes_cfg2.txt 2>&1
tail -6 gpurun_out/classes_cfg2.txt
BENCH_DEBUG=1 timeout 400 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg2.log 2> gpurun_out/bench_cfg2.err
tail -1 gpurun_out/bench_cfg2.log | cut -c 1-200
cat gpurun_out/bench_cfg2.err | tail -10
