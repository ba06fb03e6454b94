mkdir -p gpurun_out
for W in c3 c4 c5; do
  timeout 900 python bench.py --workload $W --steps 10 --warmup 3 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err; echo "$W rc=$?"
  tail -2 gpurun_out/bench_$W.err; cat gpurun_out/bench_$W.json
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -2 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
