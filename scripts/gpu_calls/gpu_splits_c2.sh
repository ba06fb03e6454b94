F="--workload c2 --no-e2e --no-cpu-baseline --no-variant --no-scan --steps 50"
for S in 4 8 12 23 37 46; do
AMS_DIAG_SPLITS=$S AMS_LIBRARY=diag_lib/libams_diag_ams_diag_splits_env.so timeout 300 python bench.py $F > gpurun_out/sp.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/sp.json').read().strip().splitlines()[-1]); r=d['roofline']; print('S=$S', d['plan'], round(r['kernel_ms_avg'],4), round(r['achieved']))"
done
