# fresh-container re-check: smoke, GPU tests, default bench, reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 180 python __graft_entry__.py smoke > gpurun_out/e_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/e_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/e_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/e_tests.log
timeout 600 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/e_bench.json default
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/e_ref.json 2> gpurun_out/e_ref.err; echo "ref rc=$?"; tail -c 400 gpurun_out/e_ref.json
