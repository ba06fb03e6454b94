timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_graphs.py tests/test_gpu_collective1.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
PYTHONPATH=. timeout 300 python scripts/debug_pair_scan.py | grep -c "bad queries 0 "
TIME=1 timeout 300 python scripts/scan_pair_calls.py
F="--no-e2e --no-cpu-baseline --no-variant --no-scan"
timeout 300 python bench.py --workload c3scan $F > gpurun_out/rg.json 2>/dev/null; python scripts/bench_summary.py gpurun_out/rg.json c3scan
timeout 300 python bench.py --workload c3scan --ungated $F > gpurun_out/rg.json 2>/dev/null; python scripts/bench_summary.py gpurun_out/rg.json c3scan-ungated
timeout 900 python bench.py --workload c5 --steps 100 > gpurun_out/rg_c5.json 2> gpurun_out/rg_c5.err; echo "c5 rc=$?"
python scripts/bench_summary.py gpurun_out/rg_c5.json c5
python -c "import json; d=json.loads(open('gpurun_out/rg_c5.json').read().strip().splitlines()[-1]); print(d['clocks'], d['latency_ms'])"
