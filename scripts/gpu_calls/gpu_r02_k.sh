# per-kernel launch times of small-batch calls (cold/serialised under ncu): where the
# non-scan time of a call goes (prep, order, merge)
set -x
i=0
for args in "c3 --nq 64 --gamma inf" "c3 --nq 64" "c3 --nq 200 --k 8" "c3 --nq 1" "c4 --nq 64" "c4 --nq 64 --gamma inf"; do
  i=$((i+1))
  python scripts/one_call.py $args --calls 5
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lt_$i.csv \
      python scripts/one_call.py $args --calls 5 > /dev/null 2>&1
  python scripts/launch_times.py gpurun_out/lt_$i.csv "$args"
done
