mkdir -p gpurun_out
python scripts/diag_power.py multicast 2>&1 | grep label
AMS_POLICY=2 python scripts/diag_power.py pair 2>&1 | grep label
python scripts/diag_power.py multicast 2>&1 | grep label
AMS_POLICY=2 python scripts/diag_power.py pair 2>&1 | grep label
F="--no-e2e --no-cpu-baseline --no-variant --no-scan"
for pol in 0 2 0 2; do
  timeout 600 python bench.py $F --kernel-policy $pol > gpurun_out/mc_b$pol.json 2> gpurun_out/mc_b$pol.err; echo "bench pol=$pol rc=$?"
  python scripts/bench_summary.py gpurun_out/mc_b$pol.json c3-pol$pol
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/mc_all.log 2>&1; echo "all tests rc=$?"; tail -3 gpurun_out/mc_all.log
