mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sorted.py tests/test_gpu_gate_first.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/2d_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/2d_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/2d_bench.json 2> gpurun_out/2d_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/2d_bench.json default
python -c "
import json; d=json.loads(open('gpurun_out/2d_bench.json').read().strip().splitlines()[-1]); print(json.dumps(d.get('gate_first_variant')))"
timeout 300 python scripts/diag_power.py product > gpurun_out/2d_pw.log 2>&1; grep label gpurun_out/2d_pw.log
