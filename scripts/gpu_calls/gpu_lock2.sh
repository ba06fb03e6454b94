mkdir -p gpurun_out
F="--no-e2e --no-cpu-baseline --no-variant --no-scan --steps 50"
for i in 1 2; do
timeout 300 python bench.py --workload c2 $F > gpurun_out/l2_p.json 2>/dev/null; python scripts/bench_summary.py gpurun_out/l2_p.json c2-product
AMS_LIBRARY=diag_lib/libams_diag_ams_diag_no_lockstep.so timeout 300 python bench.py --workload c2 $F > gpurun_out/l2_n.json 2>/dev/null; python scripts/bench_summary.py gpurun_out/l2_n.json c2-nolock
done
