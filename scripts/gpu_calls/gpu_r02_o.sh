# programmatic dependent launches (prep -> match -> merge), bounds zeroed in prep:
# full GPU suite, then in-stream timelines
set -x
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for args in "c3 --nq 64 --gamma inf" "c3 --nq 64" "c3 --nq 1" "c3 --nq 200 --k 8" "c2 --nq 4096" "c4 --nq 64"; do
  timeout 300 python scripts/one_call.py $args --calls 5 --timeline 2>&1 | grep -v "Warn\|_warn" | head -8
done
