mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sorted.py -x -q > gpurun_out/p2_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/p2_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-variant > gpurun_out/p2_bench.json 2> gpurun_out/p2_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/p2_bench.json default
B="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_c3 -f python bench.py $B > gpurun_out/p2_n2.log 2>&1; echo "full c3 rc=$?"
