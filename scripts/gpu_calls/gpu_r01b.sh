# round-1 (session 2) refresh: launch list + full ncu captures of the current kernels, nq sweep
mkdir -p gpurun_out
K='regex:match_tc|match_simt|merge_|query_prep|append_kernel|gate_scan|score_kernel'
A="--steps 2 --warmup 3"
timeout 600 python bench.py $A > gpurun_out/r1b_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_c3.csv python bench.py $A > gpurun_out/r1b_launch.log 2>&1
echo "launch rc=$?"
B="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_c3 -f python bench.py $B > gpurun_out/r1b_n2.log 2>&1
echo "full c3 rc=$?"
C="--workload c3scan --steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_scan -f python bench.py $C > gpurun_out/r1b_n3.log 2>&1
echo "full scan rc=$?"
timeout 900 python scripts/nq_sweep.py c5 > gpurun_out/sweep_c5.log 2>&1; echo "sweep c5 rc=$?"
timeout 600 python scripts/nq_sweep.py c3 > gpurun_out/sweep_c3.log 2>&1; echo "sweep c3 rc=$?"
