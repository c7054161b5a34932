(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo exit $? >> gpurun_out/gpu_tests.log)
tail -2 gpurun_out/gpu_tests.log
python scripts/batch_classes.py 2 34 > gpurun_out/classes_cfg2.txt 2>&1; head -10 gpurun_out/classes_cfg2.txt
CLASSES=1 python scripts/ncu_cfg4.py
