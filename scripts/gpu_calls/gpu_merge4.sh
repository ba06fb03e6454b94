timeout 1200 python -m pytest tests/test_gpu_scan.py tests/test_gpu_parity.py tests/test_gpu_collective1.py tests/test_gpu_graphs.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py -x -q 2>&1 | tail -2
F="--no-e2e --no-cpu-baseline --no-variant --no-scan"
for g in "" "--ungated"; do
timeout 300 python bench.py --workload c3scan $F $g > gpurun_out/m4.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/m4.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$g', d['plan'], round(d['ms_per_step'],4), round(r['kernel_ms_avg'],4), round(d['value']))"
done
