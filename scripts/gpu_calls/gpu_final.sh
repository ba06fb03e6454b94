# round-end style check: smoke, full GPU suite, default bench, reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 180 python __graft_entry__.py smoke > gpurun_out/z_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/z_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/z_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/z_tests.log
timeout 600 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/z_bench.json default
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/z_ref.json 2> gpurun_out/z_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/z_ref.json
