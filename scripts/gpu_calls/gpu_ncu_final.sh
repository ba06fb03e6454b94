mkdir -p gpurun_out
K='regex:match_tc|match_simt|merge_|query_prep|append_kernel|gate_scan|score_kernel'
A="--steps 2 --warmup 3"
python bench.py $A > gpurun_out/f_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_c3_final.csv python bench.py $A > gpurun_out/f_launch.log 2>&1
echo "launch rc=$?"
B="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
python bench.py $B > gpurun_out/f_p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_c3_final -f python bench.py $B > gpurun_out/f_n2.log 2>&1
echo "full c3 rc=$?"
C="--workload c3scan --steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
python bench.py $C > gpurun_out/f_p3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_scan_final -f python bench.py $C > gpurun_out/f_n3.log 2>&1
echo "full scan rc=$?"
D="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant --gate-first"
python bench.py $D > gpurun_out/f_p4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gate_scan -s 3 -c 1 -o gpurun_out/prof_gf_final -f python bench.py $D > gpurun_out/f_n4.log 2>&1
echo "full gf rc=$?"
