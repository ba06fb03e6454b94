# round 2: full GPU suite, smoke, compute-sanitizer on the small cases of every kernel family
set -x
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 | tee gpurun_out/r02_gputests_e.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/memcheck_cases.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.log
done
