set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
ls -la MEASURED_PEAKS.json 2>&1; cat MEASURED_PEAKS.json 2>&1 | head -40
timeout 180 python __graft_entry__.py smoke 2>&1 | tail -30
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench_default.log
