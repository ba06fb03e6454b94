# round 2: small-batch CTA-pair list write-out (skip unused lists, batched loads) -- tests + timing
set -x
timeout 1200 python -m pytest tests/test_gpu_scan.py tests/test_gpu_collective1.py -x -q 2>&1 | tail -3
timeout 600 python scripts/nq_sweep.py c3 --k 8 --nq 64,129,160,200,224,256 2>&1 | grep "gamma"
timeout 900 python scripts/nq_sweep.py c5 --nq 129,200,256 2>&1 | grep "gamma=0.3"
