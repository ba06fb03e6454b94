mkdir -p gpurun_out
N="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
timeout 600 python scripts/scan_pair_calls.py > gpurun_out/pf_pair.log 2>&1; echo "pair calls rc=$?"; tail -1 gpurun_out/pf_pair.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/pf_c3 -f python bench.py $N > gpurun_out/pf_1.log 2>&1; echo "ncu c3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/pf_c2 -f python bench.py --workload c2 $N > gpurun_out/pf_2.log 2>&1; echo "ncu c2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_scan -s 2 -c 1 -o gpurun_out/pf_pair -f python scripts/scan_pair_calls.py > gpurun_out/pf_3.log 2>&1; echo "ncu pair rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:match_|merge_|query_" --csv --log-file gpurun_out/pf_launch_c3.csv python bench.py --steps 2 --warmup 3 > gpurun_out/pf_4.log 2>&1; echo "launch c3 rc=$?"
