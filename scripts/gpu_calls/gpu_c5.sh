mkdir -p gpurun_out
timeout 900 python bench.py --workload c5 --steps 100 > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err; echo "c5 rc=$?"
python scripts/bench_summary.py gpurun_out/c5_bench.json c5
python -c "
import json; d=json.loads(open('gpurun_out/c5_bench.json').read().strip().splitlines()[-1]); print(d['clocks'], d['step_ms'], d['latency_ms'])"
timeout 900 python bench.py --workload c5 --steps 100 --gate-first > gpurun_out/c5g_bench.json 2> gpurun_out/c5g_bench.err; echo "c5g rc=$?"
python scripts/bench_summary.py gpurun_out/c5g_bench.json c5-gate-first
timeout 900 python scripts/nq_sweep.py c5 > gpurun_out/c5_sweep.log 2>&1; echo "sweep rc=$?"
