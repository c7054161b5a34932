mkdir -p gpurun_out
(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/x_tests.log 2>&1; echo exit $? >> gpurun_out/x_tests.log)
tail -3 gpurun_out/x_tests.log; grep -E "^E |FAILED" gpurun_out/x_tests.log | head -10
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python scripts/compress_time.py 2 4 2>&1 | tail -4
