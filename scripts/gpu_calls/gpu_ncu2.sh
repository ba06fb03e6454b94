mkdir -p gpurun_out
K='regex:match_tc|match_simt|merge_|query_prep|append_kernel'
A="--steps 2 --warmup 3"
python bench.py $A > gpurun_out/plain_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_c3.csv python bench.py $A > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
B="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline"
python bench.py $B > gpurun_out/plain_c3b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_c3 -f python bench.py $B > gpurun_out/ncu_full_c3.log 2>&1
echo "full c3 rc=$?"
C="--workload c3scan --steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline"
python bench.py $C > gpurun_out/plain_scan.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_scan -f python bench.py $C > gpurun_out/ncu_full_scan.log 2>&1
echo "full scan rc=$?"
