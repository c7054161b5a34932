timeout 600 compute-sanitizer --tool initcheck --print-limit 50 --error-exitcode 9 python scripts/sanitize_target.py > gpurun_out/profiles/r02_sanitizer_initcheck_after_fix.txt 2>&1; echo "initcheck exit $?"
tail -2 gpurun_out/profiles/r02_sanitizer_initcheck_after_fix.txt
bash scripts/bench_all.sh r02b
timeout 1500 python scripts/ablation_refine20.py 20 11 > gpurun_out/profiles/r02_ablation_q11.txt 2>&1; tail -3 gpurun_out/profiles/r02_ablation_q11.txt
