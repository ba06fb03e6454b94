# per-config benches + one ncu --set full capture of the match kernel per config
mkdir -p gpurun_out
F="--no-e2e --no-cpu-baseline --no-variant"
timeout 600 python bench.py --workload c2 $F > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err; echo "c2 rc=$?"
python scripts/bench_summary.py gpurun_out/f_c2.json c2
timeout 600 python bench.py --workload c3scan --ungated $F --no-scan > gpurun_out/f_scanu.json 2> gpurun_out/f_scanu.err; echo "scan-ungated rc=$?"
python scripts/bench_summary.py gpurun_out/f_scanu.json c3scan-ungated
timeout 900 python bench.py --workload c4 --steps 5 $F > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err; echo "c4 rc=$?"
python scripts/bench_summary.py gpurun_out/f_c4.json c4
timeout 900 python bench.py --workload c5 --steps 100 > gpurun_out/f_c5.json 2> gpurun_out/f_c5.err; echo "c5 rc=$?"
python scripts/bench_summary.py gpurun_out/f_c5.json c5
N="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_c2 -f python bench.py --workload c2 $N > gpurun_out/f_n2.log 2>&1; echo "full c2 rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_c4 -f python bench.py --workload c4 $N > gpurun_out/f_n4.log 2>&1; echo "full c4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:match_tc|merge_|query_|append_kernel" --csv --log-file gpurun_out/launches_c5.csv python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/f_l5.log 2>&1; echo "launch c5 rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 40 -c 1 -o gpurun_out/prof_c5 -f python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/f_n5.log 2>&1; echo "full c5 rc=$?"
