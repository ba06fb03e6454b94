mkdir -p gpurun_out
K='regex:match_tc|match_simt|merge_|query_prep|query_order|append_kernel|gate_scan|score_kernel'
A="--steps 2 --warmup 3"
timeout 600 python bench.py $A > gpurun_out/r1d_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_c3.csv python bench.py $A > gpurun_out/r1d_launch.log 2>&1
echo "launch rc=$?"
for W in c4 c2 c5; do
  timeout 900 python bench.py --workload $W --no-cpu-baseline > gpurun_out/r1d_$W.json 2> gpurun_out/r1d_$W.err; echo "$W rc=$?"
  python scripts/bench_summary.py gpurun_out/r1d_$W.json $W
done
timeout 600 python bench.py --workload c3 --ungated --no-cpu-baseline > gpurun_out/r1d_c3u.json 2> gpurun_out/r1d_c3u.err; echo "c3u rc=$?"
python scripts/bench_summary.py gpurun_out/r1d_c3u.json c3u
