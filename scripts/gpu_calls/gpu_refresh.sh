mkdir -p gpurun_out
F="--no-e2e --no-cpu-baseline --no-variant --no-scan"
timeout 300 python bench.py --workload c2 $F --steps 50 > gpurun_out/r_c2.json 2>/dev/null; python scripts/bench_summary.py gpurun_out/r_c2.json c2
timeout 300 python bench.py --workload c2 $F --steps 50 --ungated > gpurun_out/r_c2u.json 2>/dev/null; python scripts/bench_summary.py gpurun_out/r_c2u.json c2-ungated
timeout 300 python bench.py $F > gpurun_out/r_c3.json 2>/dev/null; python scripts/bench_summary.py gpurun_out/r_c3.json c3
timeout 300 python bench.py $F --ungated > gpurun_out/r_c3u.json 2>/dev/null; python scripts/bench_summary.py gpurun_out/r_c3u.json c3-ungated
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sorted.py tests/test_gpu_fullsize.py tests/test_gpu_multicast.py -x -q 2>&1 | tail -2
