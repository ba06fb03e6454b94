timeout 600 python -m pytest tests/test_gpu_graphs.py -x -q 2>&1 | tail -15
timeout 300 python scripts/graph_latency.py
