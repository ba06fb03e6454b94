timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_graphs.py tests/test_gpu_collective1.py tests/test_gpu_sharding.py -x -q 2>&1 | tail -3
timeout 300 python scripts/graph_latency.py
timeout 300 ncu --metrics gpu__time_duration.sum --csv --clock-control none python scripts/c1_calls.py 2>/dev/null > gpurun_out/c1_launch2.csv
