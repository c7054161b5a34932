timeout 1500 python scripts/ablation_refine20.py 24 > gpurun_out/ablation20.txt 2>&1; tail -30 gpurun_out/ablation20.txt
