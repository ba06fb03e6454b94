# rank-based block merge: full GPU suite and in-stream timelines
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k block_merge 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for args in "c3 --nq 64 --gamma inf" "c3 --nq 64" "c3 --nq 1" "c4 --nq 64 --gamma inf" "c4 --nq 64"; do
  timeout 300 python scripts/one_call.py $args --calls 5 --timeline 2>&1 | grep -v Warn | head -9
done
