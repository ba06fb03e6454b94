# full GPU suite, default bench, ncu captures of the small-batch kernel (C3 scan gated/ungated, C5)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/g_tests.log
timeout 600 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/g_bench.json default
N="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_scan -s 3 -c 1 -o gpurun_out/prof_scan_g -f python bench.py --workload c3scan $N > gpurun_out/g_n1.log 2>&1; echo "ncu scan rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_scan -s 3 -c 1 -o gpurun_out/prof_scanu_g -f python bench.py --workload c3scan --ungated $N > gpurun_out/g_n2.log 2>&1; echo "ncu scan-ungated rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:match_|merge_|query_|append_kernel" --csv --log-file gpurun_out/launches_c5g.csv python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/g_l5.log 2>&1; echo "launch c5 rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:match_scan -s 40 -c 1 -o gpurun_out/prof_c5_g -f python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/g_n5.log 2>&1; echo "ncu c5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:match_|merge_|query_" --csv --log-file gpurun_out/launches_c3g.csv python bench.py --steps 2 --warmup 3 > gpurun_out/g_l3.log 2>&1; echo "launch c3 rc=$?"
