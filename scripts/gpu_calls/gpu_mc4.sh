mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multicast.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_sorted.py -x -q > gpurun_out/mc4_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/mc4_tests.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-variant > gpurun_out/mc4_b.json 2> gpurun_out/mc4_b.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/mc4_b.json default
