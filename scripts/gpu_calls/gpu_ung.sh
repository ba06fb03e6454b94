mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py tests/test_gpu_sorted.py tests/test_gpu_sharding.py -x -q > gpurun_out/ung_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/ung_tests.log
timeout 600 python bench.py --ungated --no-cpu-baseline --no-variant > gpurun_out/ung_bench.json 2> gpurun_out/ung_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/ung_bench.json ungated
timeout 600 python bench.py --no-cpu-baseline --no-variant > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/g_bench.json gated
timeout 300 python scripts/diag_power.py product > gpurun_out/pw2_product.log 2>&1; grep label gpurun_out/pw2_product.log
timeout 600 python scripts/nq_sweep.py c3 > gpurun_out/ung_sweep_c3.log 2>&1; echo "sweep rc=$?"
