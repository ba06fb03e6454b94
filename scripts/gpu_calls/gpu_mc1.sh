mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_multicast.py -x -q > gpurun_out/mc_tests.log 2>&1; echo "mc tests rc=$?"; tail -15 gpurun_out/mc_tests.log
nvidia-smi --query-gpu=name,utilization.gpu --format=csv
