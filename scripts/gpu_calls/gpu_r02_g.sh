# round 2: MMA N = round_up(nq, 16) in the small-batch kernel -- scan/parity tests and the nq sweeps
set -x
timeout 1200 python -m pytest tests/test_gpu_scan.py tests/test_gpu_parity.py tests/test_gpu_sorted.py tests/test_gpu_edge.py tests/test_gpu_graphs.py -x -q 2>&1 | tail -6
timeout 600 python scripts/nq_sweep.py c3 --k 8 --nq 1,16,17,33,64,100,129,144,160,200,208,224,256 2>&1 | grep "gamma=0.3"
timeout 900 python scripts/nq_sweep.py c5 --nq 1,17,64,100,129,200,256 2>&1 | grep "gamma=0.3"
