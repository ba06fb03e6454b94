# L2 reuse vs unit length: DRAM bytes of match_tc on C4/C3 with S x {1,2,4,8} (diag builds)
mkdir -p gpurun_out
M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second
for W in c4 c3; do
  for m in 1 2 4 8; do
    if [ $m = 1 ]; then unset AMS_LIBRARY; else export AMS_LIBRARY=$PWD/diag_lib/libams_diag_ams_diag_split_mult_$m.so; fi
    B="--workload $W --steps 3 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
    python bench.py $B > gpurun_out/sp_${W}_$m.json 2> gpurun_out/sp_${W}_$m.err
    ncu --metrics $M --clock-control none -k regex:match_tc -s 3 -c 1 --csv python bench.py $B > gpurun_out/spn_${W}_$m.csv 2> gpurun_out/spn_${W}_$m.err
    echo "$W x$m rc=$?"
  done
done
