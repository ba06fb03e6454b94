mkdir -p gpurun_out
M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second
B="--steps 10 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
for m in 1 2 4; do
  if [ $m = 1 ]; then unset AMS_LIBRARY; else export AMS_LIBRARY=$PWD/diag_lib/libams_diag_ams_diag_split_mult_$m.so; fi
  timeout 600 python bench.py $B > gpurun_out/sp2_$m.json 2> gpurun_out/sp2_$m.err
  python scripts/bench_summary.py gpurun_out/sp2_$m.json x$m
  timeout 600 ncu --metrics $M --clock-control none -k regex:match_tc -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant > gpurun_out/sp2n_$m.csv 2> gpurun_out/sp2n_$m.err
  grep -E "dram__bytes_read|gpu__time_duration|hit_rate" gpurun_out/sp2n_$m.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
