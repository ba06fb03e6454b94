# ncu source-level capture of the merge after an ungated 64-query C3 scan (warm L2, as in-stream)
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:merge_partials --launch-skip 3 -c 1 \
   -o gpurun_out/ncu_merge_ungated -f python scripts/one_call.py c3 --nq 64 --gamma inf --calls 5 > gpurun_out/ncu_merge.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_merge.log
