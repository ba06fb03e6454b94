# round 2: wide small-batch CTA pairs -- parity (scan tests) and the 129-256-query timing, wide vs narrow
set -x
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_vstore.py -x -q 2>&1 | tail -12
for pol in 0 4; do timeout 600 python scripts/nq_sweep.py c3 --k 8 --policy $pol --nq 64,129,160,200,224,256 2>&1 | grep "gamma=0.3" ; done
for pol in 0 4; do timeout 900 python scripts/nq_sweep.py c5 --policy $pol --nq 64,129,200,256 2>&1 | grep "gamma=0.3" ; done
