timeout 600 python -m pytest tests/test_gpu_hash.py tests/test_gpu_vstore.py -x -q 2>&1 | tail -2
timeout 300 python scripts/hash_speed.py
timeout 300 python scripts/hash_speed.py
