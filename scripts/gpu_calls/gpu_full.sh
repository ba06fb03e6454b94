# full check: GPU tests, default bench, small-batch launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/fu_tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/fu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/fu_bench.json 2> gpurun_out/fu_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/fu_bench.json default
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:match_tc|merge_|query_" --csv python scripts/small_nq.py > gpurun_out/fu_small_nq.csv 2> gpurun_out/fu_small_nq.err; echo "ncu rc=$?"
