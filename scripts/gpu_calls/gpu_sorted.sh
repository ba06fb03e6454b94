mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sorted.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -x -q > gpurun_out/so_tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/so_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/so_bench.json 2> gpurun_out/so_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/so_bench.json 2>&1 | tail -5
timeout 900 python scripts/nq_sweep.py c5 > gpurun_out/so_sweep_c5.log 2>&1; echo "sweep rc=$?"
