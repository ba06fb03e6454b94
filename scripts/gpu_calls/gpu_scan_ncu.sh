mkdir -p gpurun_out
N="--steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_scan -s 3 -c 1 -o gpurun_out/prof_scanu_new -f python bench.py --workload c3scan --ungated $N > gpurun_out/sn1.log 2>&1; echo "ncu ungated rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_scan -s 3 -c 1 -o gpurun_out/prof_scan_new -f python bench.py --workload c3scan $N > gpurun_out/sn2.log 2>&1; echo "ncu gated rc=$?"
