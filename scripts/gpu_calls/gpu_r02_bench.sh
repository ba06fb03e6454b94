# the driver's default bench command on the current build (ncu_summary.json already holds this build's captures)
set -x
python -c "import paper_2508_10259_b200 as a; print(a.ams_build_id())"
timeout 1200 python bench.py > gpurun_out/r02_bench_final3.json 2> gpurun_out/r02_bench_final3.err; echo "bench rc=$?"
