# binned gate-first for every gated batch > 16 queries: tests, then timelines incl. the C3 batch
set -x
timeout 1500 python -m pytest tests/test_gpu_gate_first.py tests/test_gpu_auto.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -3
for args in "c3 --nq 1024 --gate-first" "c3 --nq 4096 --gate-first" "c3 --nq 16384 --gate-first" "c5 --nq 256 --auto"; do
  timeout 400 python scripts/one_call.py $args --calls 5 --timeline 2>&1 | grep -v "Warn\|_warn" | head -7
done
