# round 2 profile refresh: default bench line, launch list of the bench command, ncu --set full
# of the dominant kernels (C3 batch K2, C3 64-query scan K2s, hash TC, C4 batch K2) with the
# library's build id recorded next to the reports (bench.py reuses the traffic only for that build)
set -x
python -c "import paper_2508_10259_b200 as a; print(a.ams_build_id())" > gpurun_out/prof_buildid.txt
timeout 1200 python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err; echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02_c3.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c4 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc_kernel -c 1 \
   -o gpurun_out/ncu_r02_c3_match_tc -f python scripts/one_call.py c3 --nq 16384 --k 16 --calls 1 > gpurun_out/ncu_k2.log 2>&1; echo "k2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_scan_kernel --launch-skip 3 -c 1 \
   -o gpurun_out/ncu_r02_c3_match_scan -f python scripts/one_call.py c3 --nq 64 --k 16 > gpurun_out/ncu_k2s.log 2>&1; echo "k2s rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_scan_kernel --launch-skip 3 -c 1 \
   -o gpurun_out/ncu_r02_c3_200q_k8_pair -f python scripts/one_call.py c3 --nq 200 --k 8 > gpurun_out/ncu_pair.log 2>&1; echo "pair rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:phase1_tc_kernel -c 1 \
   -o gpurun_out/ncu_r02_hash_phase1_tc -f python scripts/hash_speed.py > gpurun_out/ncu_hash2.log 2>&1; echo "hash rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gate_rows_snap --launch-skip 3 -c 1 \
   -o gpurun_out/ncu_r02_c5_64q_gate_rows_snap -f python scripts/one_call.py c5 --nq 64 --gate-first > gpurun_out/ncu_gsnap.log 2>&1; echo "gsnap rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --steps 10 --warmup 3 --force-collective --no-cpu-baseline > gpurun_out/r02_dry_collective2.json 2> gpurun_out/r02_dry_collective2.err
echo "dry rc=$?"
