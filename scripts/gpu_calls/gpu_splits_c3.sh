F="--no-e2e --no-cpu-baseline --no-variant --no-scan --steps 10"
for S in 37 74 111 148; do
AMS_DIAG_SPLITS=$S AMS_LIBRARY=diag_lib/libams_diag_ams_diag_splits_env.so timeout 300 python bench.py $F > gpurun_out/sp3.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/sp3.json').read().strip().splitlines()[-1]); r=d['roofline']; print('S=$S', d['plan'], round(r['kernel_ms_avg'],3), round(r['achieved']), round(d['ms_per_step'],3))"
AMS_DIAG_SPLITS=$S AMS_LIBRARY=diag_lib/libams_diag_ams_diag_splits_env.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:match_tc -s 3 -c 1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-variant --no-scan 2>/dev/null | grep -E "dram__bytes|gpu__time"
done
