# GPU parity suite + smoke; logs under gpurun_out/.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash scripts/gpu_tests.sh [pytest args]'
(timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/gpu_tests.log 2>&1; echo exit $? >> gpurun_out/gpu_tests.log)
tail -15 gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
