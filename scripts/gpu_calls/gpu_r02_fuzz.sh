# a long randomized differential sweep (seeded; expected values from oracle/ only)
set -x
AMS_FUZZ_CASES=800 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -q -x 2>&1 | tail -8
