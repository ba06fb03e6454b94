mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gate_first.py tests/test_gpu_sorted.py -x -q > gpurun_out/gf_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gf_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-scan > gpurun_out/gf_bench.json 2> gpurun_out/gf_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/gf_bench.json').read().strip().splitlines()[-1]); print(d['value'], json.dumps(d.get('gate_first_variant')))"
