mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sorted.py tests/test_gpu_gate_first.py -x -q > gpurun_out/so2_tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/so2_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/so2_bench.json 2> gpurun_out/so2_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/so2_bench.json 2>&1 | tail -5
python -c "
import json; d=json.loads(open('gpurun_out/so2_bench.json').read().strip().splitlines()[-1]); print(json.dumps(d.get('gate_first_variant')))"
