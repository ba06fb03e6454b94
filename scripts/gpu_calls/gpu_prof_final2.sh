mkdir -p gpurun_out
N="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_scan -s 3 -c 1 -o gpurun_out/fz_scan -f python bench.py --workload c3scan $N > /dev/null 2>&1; echo "scan rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_scan -s 2 -c 1 -o gpurun_out/fz_pair -f python scripts/scan_pair_calls.py > /dev/null 2>&1; echo "pair rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:match_|merge_|query_|append_kernel" --csv --log-file gpurun_out/fz_launch_c5.csv python bench.py --workload c5 --steps 5 --warmup 3 > /dev/null 2>&1; echo "launch c5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:match_|merge_|query_" --csv --log-file gpurun_out/fz_launch_c3.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1; echo "launch c3 rc=$?"
