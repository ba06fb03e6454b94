# round 2: tensor-core hash path (tests, speed, ncu), auto-route tests
set -x
timeout 900 python -m pytest tests/test_gpu_hash.py tests/test_gpu_auto.py tests/test_gpu_vstore.py -x -q 2>&1 | tail -15
timeout 300 python scripts/hash_speed.py 2>&1 | tail -5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:phase1_tc_kernel -c 1 -o gpurun_out/ncu_r02_hash_tc -f python scripts/hash_speed.py > gpurun_out/ncu_hash.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_hash.log
