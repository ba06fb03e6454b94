# small-batch kernel: parity tests first, then A/B benches (scan, C5 streaming)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py -x -q > gpurun_out/s_tests.log 2>&1; echo "scan tests rc=$?"; tail -15 gpurun_out/s_tests.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s_all.log 2>&1; echo "all gpu tests rc=$?"; tail -15 gpurun_out/s_all.log
F="--no-e2e --no-cpu-baseline --no-variant --no-scan"
for pol in 0 1; do
  timeout 600 python bench.py --workload c3scan $F --kernel-policy $pol > gpurun_out/s_scan$pol.json 2> gpurun_out/s_scan$pol.err; echo "c3scan pol=$pol rc=$?"
  python scripts/bench_summary.py gpurun_out/s_scan$pol.json c3scan-pol$pol
  timeout 600 python bench.py --workload c3scan --ungated $F --kernel-policy $pol > gpurun_out/s_scanu$pol.json 2> gpurun_out/s_scanu$pol.err; echo "c3scan-ung pol=$pol rc=$?"
  python scripts/bench_summary.py gpurun_out/s_scanu$pol.json c3scan-ungated-pol$pol
done
for pol in 0 1; do
  timeout 900 python bench.py --workload c5 --steps 100 --kernel-policy $pol > gpurun_out/s_c5_$pol.json 2> gpurun_out/s_c5_$pol.err; echo "c5 pol=$pol rc=$?"
  python scripts/bench_summary.py gpurun_out/s_c5_$pol.json c5-pol$pol
  python -c "import json; d=json.loads(open('gpurun_out/s_c5_$pol.json').read().strip().splitlines()[-1]); print(d['clocks'], d['latency_ms'])"
done
