# full GPU suite on the current build, smoke, and a 400-case fuzz sweep
set -x
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
AMS_FUZZ_CASES=400 timeout 1500 python -m pytest tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
