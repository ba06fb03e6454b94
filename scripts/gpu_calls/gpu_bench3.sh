mkdir -p gpurun_out
for A in "--workload c3" "--workload c3 --ungated" "--workload c4" "--workload c4 --ungated"; do
  timeout 900 python bench.py $A --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b3.json 2> gpurun_out/b3.err; echo "$A rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/b3.json'))
print('value %.0f q/s  kern %.2f ms  %.0f TF frac %.3f  clocks %s  scan %.0f GB/s frac %.3f' % (d['value'], d['roofline']['kernel_ms_avg'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'], d['scan']['roofline']['achieved'], d['scan']['roofline']['frac']))"
done
