mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py -x -q > gpurun_out/wv_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/wv_tests.log
M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second
for W in c4 c3; do
  B="--workload $W --steps 3 --warmup 3 --no-scan --no-e2e --no-cpu-baseline --no-variant"
  timeout 600 python bench.py $B > gpurun_out/wv_${W}.json 2> gpurun_out/wv_${W}.err
  echo "$W bench rc=$?"
  timeout 600 ncu --metrics $M --clock-control none -k regex:match_tc -s 3 -c 1 --csv python bench.py $B > gpurun_out/wvn_${W}.csv 2> gpurun_out/wvn_${W}.err
  echo "$W ncu rc=$?"
  AMS_LIBRARY=$PWD/diag_lib/libams_diag_ams_diag_timeline.so timeout 600 python scripts/diag_timeline.py $W gpurun_out/tlw_$W.npz 2>&1 | tail -1
done
