PYTHONPATH=. timeout 300 python scripts/debug_pair_scan.py | grep -c "bad queries 0 "
TIME=1 timeout 300 python scripts/scan_pair_calls.py
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_collective1.py -x -q 2>&1 | tail -2
