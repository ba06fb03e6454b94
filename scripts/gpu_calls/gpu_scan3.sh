mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_large.py -x -q > gpurun_out/s3_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_tests.log
F="--no-e2e --no-cpu-baseline --no-variant --no-scan"
for pol in 0 1; do
  timeout 900 python bench.py --workload c4 --steps 5 --no-e2e --no-cpu-baseline --no-variant --kernel-policy $pol > gpurun_out/s3_c4_$pol.json 2> gpurun_out/s3_c4_$pol.err; echo "c4 pol=$pol rc=$?"
  python scripts/bench_summary.py gpurun_out/s3_c4_$pol.json c4-pol$pol
  timeout 600 python bench.py --workload c3scan $F --kernel-policy $pol > gpurun_out/s3_scan$pol.json 2> gpurun_out/s3_scan$pol.err; echo "c3scan pol=$pol rc=$?"
  python scripts/bench_summary.py gpurun_out/s3_scan$pol.json c3scan-pol$pol
done
