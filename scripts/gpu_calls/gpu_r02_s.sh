# ncu of the warp-per-query merge after a C2 batch (4096 queries, 46 lists per query)
set -x
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:merge_partials --launch-skip 3 -c 1 \
   -o gpurun_out/ncu_merge_c2 -f python scripts/one_call.py c2 --nq 4096 --calls 5 > gpurun_out/ncu_merge_c2.log 2>&1
echo "rc=$?"
