mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/s2_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/s2_tests.log
F="--no-e2e --no-cpu-baseline --no-variant --no-scan"
for pol in 0 1; do
  timeout 600 python bench.py --workload c3scan --ungated $F --kernel-policy $pol > gpurun_out/s2_scanu$pol.json 2> gpurun_out/s2_scanu$pol.err; echo "c3scan-ung pol=$pol rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/s2_scanu$pol.json').read().strip().splitlines()[-1]); r=d['roofline']; print($pol, round(d['ms_per_step'],4), round(r['kernel_ms_avg'],4), round(r['frac'],3))"
done
timeout 600 python bench.py --workload c3scan $F > gpurun_out/s2_scan0.json 2> gpurun_out/s2_scan0.err; echo "c3scan rc=$?"
python scripts/bench_summary.py gpurun_out/s2_scan0.json c3scan
