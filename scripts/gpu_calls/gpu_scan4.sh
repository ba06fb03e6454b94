mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py -x -q > gpurun_out/s4_tests.log 2>&1; echo "scan tests rc=$?"; tail -15 gpurun_out/s4_tests.log
timeout 900 python bench.py --workload c5 --steps 100 > gpurun_out/s4_c5.json 2> gpurun_out/s4_c5.err; echo "c5 rc=$?"
python scripts/bench_summary.py gpurun_out/s4_c5.json c5
python -c "import json; d=json.loads(open('gpurun_out/s4_c5.json').read().strip().splitlines()[-1]); print(d['clocks'], d['latency_ms'])"
