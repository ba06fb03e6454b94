# gate-first snapshot-window kernel with the next row group's joints loaded ahead: tests, timelines
set -x
timeout 1200 python -m pytest tests/test_gpu_gate_first.py tests/test_gpu_auto.py -x -q 2>&1 | tail -2
for args in "c3 --nq 64 --gate-first" "c3 --nq 200 --gate-first" "c3 --nq 1024 --gate-first" "c5 --nq 17 --auto" "c5 --nq 64 --auto" "c5 --nq 256 --auto"; do
  timeout 400 python scripts/one_call.py $args --calls 5 --timeline 2>&1 | grep -v "_warn" | head -5
done
