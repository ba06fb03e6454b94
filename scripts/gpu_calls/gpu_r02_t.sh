# ncu of the gate scan (C5 pool, 256 queries: QT = 256) and (C5 pool, 64 queries: QT = 64)
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gate_scan --launch-skip 3 -c 1 \
   -o gpurun_out/ncu_gate_c5_256 -f python scripts/one_call.py c5 --nq 256 --gate-first --calls 5 > gpurun_out/ncu_gate1.log 2>&1
echo "rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gate_scan --launch-skip 3 -c 1 \
   -o gpurun_out/ncu_gate_c5_64 -f python scripts/one_call.py c5 --nq 64 --gate-first --calls 5 > gpurun_out/ncu_gate2.log 2>&1
echo "rc=$?"
