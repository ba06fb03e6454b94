mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_sharding.py tests/test_gpu_sorted.py tests/test_gpu_exchange.py tests/test_gpu_gate_first.py -x -q > gpurun_out/mg_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/mg_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:match_tc|merge_|query_" --csv python scripts/small_nq.py > gpurun_out/mg_small_nq.csv 2> gpurun_out/mg_small_nq.err; echo "ncu rc=$?"
timeout 600 python scripts/nq_sweep.py c3 > gpurun_out/mg_sweep_c3.log 2>&1; echo "sweep rc=$?"
