mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py tests/test_gpu_sorted.py tests/test_gpu_sharding.py -x -q > gpurun_out/mma_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/mma_tests.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-variant > gpurun_out/mma_bench.json 2> gpurun_out/mma_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/mma_bench.json default
done
timeout 300 python scripts/diag_power.py product > gpurun_out/mma_pw.log 2>&1; grep label gpurun_out/mma_pw.log
timeout 600 python bench.py --workload c4 --steps 5 --no-cpu-baseline --no-e2e --no-variant --no-scan > gpurun_out/mma_c4.json 2> gpurun_out/mma_c4.err; python scripts/bench_summary.py gpurun_out/mma_c4.json c4
