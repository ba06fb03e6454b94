# round-end style check + profile refresh
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 180 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rd_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/rd_tests.log
timeout 600 python bench.py > gpurun_out/rd_bench.json 2> gpurun_out/rd_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/rd_bench.json default
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/rd_ref.json 2> gpurun_out/rd_ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/rd_ref.json
K='regex:match_tc|match_simt|merge_|query_prep|query_order|append_kernel|gate_scan|score_kernel'
A="--steps 2 --warmup 3"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_c3.csv python bench.py $A > gpurun_out/rd_launch.log 2>&1; echo "launch rc=$?"
B="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_c3 -f python bench.py $B > gpurun_out/rd_n2.log 2>&1; echo "full c3 rc=$?"
C="--workload c3scan --steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_scan -f python bench.py $C > gpurun_out/rd_n3.log 2>&1; echo "full scan rc=$?"
D="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant --gate-first"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gate_scan -s 3 -c 1 -o gpurun_out/prof_gf -f python bench.py $D > gpurun_out/rd_n4.log 2>&1; echo "full gf rc=$?"
