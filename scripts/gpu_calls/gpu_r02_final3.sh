# end-of-round check on the final build: full GPU suite, smoke, then the profile captures
# (the bench line is taken in a second call, after ncu_summary.json holds these captures)
set -x
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
cp gpurun_out/parity_tight_report.json gpurun_out/parity_tight_full_final.json
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/gpu_calls/gpu_r02_prof.sh
