# DRAM traffic / L2 hit rate of the dense match kernel on C3 and C4 (one launch each)
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read.sum
for W in c3 c4; do
  B="--workload $W --steps 1 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
  ncu --metrics $M --clock-control none -k regex:match_tc -s 3 -c 1 --csv python bench.py $B > gpurun_out/l2_$W.csv 2> gpurun_out/l2_$W.err
  echo "$W rc=$?"
done
python bench.py --steps 5 --warmup 3 --no-scan --no-variant > gpurun_out/cal.json 2> gpurun_out/cal.err
echo "cal rc=$?"
