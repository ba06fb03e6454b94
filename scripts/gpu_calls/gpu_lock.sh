mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k self_match 2>&1 | tail -2
for W in c3 c4; do
for v in prod nolock prod nolock; do
  if [ $v = prod ]; then unset AMS_LIBRARY; else export AMS_LIBRARY=$PWD/diag_lib/libams_diag_ams_diag_no_lockstep.so; fi
  timeout 600 python bench.py --workload $W --steps 10 --no-cpu-baseline --no-e2e --no-variant --no-scan > gpurun_out/lk.json 2> gpurun_out/lk.err
  python scripts/bench_summary.py gpurun_out/lk.json $W-$v
done
done
