mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5_tests.log 2>&1; echo "all tests rc=$?"; tail -15 gpurun_out/s5_tests.log
for pol in 0 1; do
timeout 900 python bench.py --workload c5 --steps 100 --kernel-policy $pol > gpurun_out/s5_c5_$pol.json 2> gpurun_out/s5_c5_$pol.err; echo "c5 rc=$?"
python scripts/bench_summary.py gpurun_out/s5_c5_$pol.json c5-pol$pol
python -c "import json; d=json.loads(open('gpurun_out/s5_c5_$pol.json').read().strip().splitlines()[-1]); print(d['clocks'], d['latency_ms'], d['step_ms'])"
done
