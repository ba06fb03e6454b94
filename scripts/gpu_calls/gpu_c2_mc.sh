F="--workload c2 --no-e2e --no-cpu-baseline --no-variant --no-scan --steps 50"
for pol in 0 2 0 2; do
timeout 300 python bench.py $F --kernel-policy $pol > gpurun_out/c2mc.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/c2mc.json').read().strip().splitlines()[-1]); r=d['roofline']; print('pol=$pol', d['plan'], round(r['kernel_ms_avg'],4), round(r['achieved']))"
done
