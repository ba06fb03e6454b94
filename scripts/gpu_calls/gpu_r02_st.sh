# CTA pairs with a single-buffered aux ring and up to 8 stages (a build reverted after this run:
# slower): scan tests, then the 129-256 band
set -x
timeout 900 python -m pytest tests/test_gpu_scan.py -x -q 2>&1 | tail -2
timeout 600 python scripts/nq_sweep.py c3 --k 8 --nq 64,129,144,160,200,208,224,256 | grep gamma=0.3
timeout 900 python scripts/nq_sweep.py c5 --nq 64,129,200,256 | grep gamma=0.3
