# ncu of the binned gate row kernel (C5 pool, 64 queries)
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gate_rows_binned --launch-skip 3 -c 1 \
   -o gpurun_out/ncu_gate_binned_c5_64 -f python scripts/one_call.py c5 --nq 64 --gate-first --calls 5 > gpurun_out/ncu_gb.log 2>&1
echo "rc=$?"
