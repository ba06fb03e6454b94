set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 180 python __graft_entry__.py smoke 2>&1 | tail -30
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
