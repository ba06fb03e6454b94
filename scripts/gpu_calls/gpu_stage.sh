mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/st_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/st_tests.log
timeout 600 python bench.py > gpurun_out/st_bench.json 2> gpurun_out/st_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/st_bench.json default
python -c "
import json; d=json.loads(open('gpurun_out/st_bench.json').read().strip().splitlines()[-1]); print(d['e2e'], d['cpu_baseline'], d['gpu_launches'])"
