# gate-first after the row-kernel fix: gate-first / auto / fuzz suites, then the whole GPU suite
set -x
timeout 1500 python -m pytest tests/test_gpu_gate_first.py tests/test_gpu_auto.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -3
AMS_FUZZ_CASES=400 timeout 1500 python -m pytest tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
