# Per-class kernel time of the cfg2 batch (bench slicing) and of the cfg4 joins.
#   /usr/local/graft/bin/gpurun --timeout 1500 -- 'bash scripts/gpu_diag.sh'
python scripts/batch_classes.py 2 34
CLASSES=1 python scripts/ncu_cfg4.py
