mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py tests/test_gpu_sorted.py tests/test_gpu_sharding.py -x -q > gpurun_out/sl_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/sl_tests.log
timeout 600 python bench.py --ungated --no-cpu-baseline --no-variant --no-e2e > gpurun_out/sl_bench.json 2> gpurun_out/sl_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/sl_bench.json ungated
timeout 600 python bench.py --no-cpu-baseline --no-variant --no-e2e > gpurun_out/sl_gbench.json 2> gpurun_out/sl_gbench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/sl_gbench.json gated
timeout 600 python scripts/nq_sweep.py c3 > gpurun_out/sl_sweep_c3.log 2>&1; echo "sweep rc=$?"
grep "gamma=inf" gpurun_out/sl_sweep_c3.log | cut -c1-60
