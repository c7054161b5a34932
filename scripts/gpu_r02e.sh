mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "torch_caching or kernel_variants or cfg2_match_batch" > gpurun_out/e_tests.log 2>&1; echo exit $? >> gpurun_out/e_tests.log)
tail -3 gpurun_out/e_tests.log; grep -E "^E |FAILED|Error" gpurun_out/e_tests.log | head -10
bash scripts/bench_all.sh r02e
