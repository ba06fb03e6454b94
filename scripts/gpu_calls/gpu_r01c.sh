mkdir -p gpurun_out
B="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -o gpurun_out/prof_c3_sorted -f python bench.py $B > gpurun_out/r1c_n.log 2>&1
echo "full c3 rc=$?"
timeout 300 python scripts/diag_power.py cublas > gpurun_out/pw_cublas.log 2>&1
timeout 300 python scripts/diag_power.py product > gpurun_out/pw_product.log 2>&1
AMS_LIBRARY=$PWD/diag_lib/libams_diag_ams_diag_no_epilogue.so timeout 300 python scripts/diag_power.py noepi > gpurun_out/pw_noepi.log 2>&1
timeout 300 python scripts/diag_power.py cublas > gpurun_out/pw_cublas2.log 2>&1
grep -h label gpurun_out/pw_*.log
