(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo exit $? >> gpurun_out/gpu_tests.log)
tail -2 gpurun_out/gpu_tests.log
python scripts/batch_classes.py 2 25 > gpurun_out/classes_cfg2.txt 2>&1
head -12 gpurun_out/classes_cfg2.txt
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1
tail -1 gpurun_out/bench_cfg2.log | cut -c 1-200
timeout 600 python bench.py --config 4 --steps 5 > gpurun_out/bench_cfg4.log 2>&1
tail -1 gpurun_out/bench_cfg4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'])"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__registers_per_thread,smsp__inst_executed.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__thread_inst_executed_per_inst_executed.ratio
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_join_fast" -c 4 -o /tmp/prof_c4 python scripts/ncu_cfg4.py > gpurun_out/ncu_c4.log 2>&1
ncu -i /tmp/prof_c4.ncu-rep --page raw --csv --metrics $M > gpurun_out/c4_raw.csv
python scripts/ncu_lines.py /tmp/prof_c4.ncu-rep gpurun_out/c4_lines 4
du -sh gpurun_out
