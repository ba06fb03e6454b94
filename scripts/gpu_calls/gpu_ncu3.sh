mkdir -p gpurun_out
B="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline"
python bench.py $B > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_c3_v2 -f python bench.py $B > gpurun_out/n1.log 2>&1
echo "full rc=$?"
export AMS_LIBRARY=$PWD/diag_lib/libams_diag.so
python bench.py $B > gpurun_out/p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_c3_noepi -f python bench.py $B > gpurun_out/n2.log 2>&1
echo "noepi rc=$?"
