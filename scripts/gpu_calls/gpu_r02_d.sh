# round 2: ncu of the small-batch CTA-pair kernel, wide (policy 0) vs narrow (policy 4), C3 pool, 200 queries, k = 8
set -x
for pol in 0 4; do
  timeout 300 python scripts/one_call.py c3 --nq 200 --k 8 --policy $pol
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_scan_kernel --launch-skip 3 -c 1 \
     -o gpurun_out/ncu_r02_pair_p$pol -f python scripts/one_call.py c3 --nq 200 --k 8 --policy $pol > gpurun_out/ncu_pair_p$pol.log 2>&1
  echo "ncu rc=$?"
done
