mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "rc=$?"
tail -3 gpurun_out/bench_c3.err
cat gpurun_out/bench_c3.json
timeout 300 python bench.py --steps 10 --warmup 3 --ungated --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_ungated.json 2> gpurun_out/bench_c3_ungated.err; echo "rc=$?"
tail -3 gpurun_out/bench_c3_ungated.err
cat gpurun_out/bench_c3_ungated.json
