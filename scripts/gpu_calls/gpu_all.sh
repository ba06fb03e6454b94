mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/all_tests.log 2>&1; echo "all tests rc=$?"; tail -4 gpurun_out/all_tests.log
timeout 180 python __graft_entry__.py smoke 2>&1 | tail -1
