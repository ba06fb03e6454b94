# final bench lines of every workload (committed as profiles/bench_r01_final.jsonl)
mkdir -p gpurun_out
rm -f gpurun_out/bench_all.jsonl
timeout 600 python bench.py 2>/dev/null | tail -1 >> gpurun_out/bench_all.jsonl; echo "c3 rc=$?"
timeout 600 python bench.py --workload c2 2>/dev/null | tail -1 >> gpurun_out/bench_all.jsonl; echo "c2 rc=$?"
timeout 600 python bench.py --workload c3scan --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/bench_all.jsonl; echo "c3scan rc=$?"
timeout 900 python bench.py --workload c4 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/bench_all.jsonl; echo "c4 rc=$?"
timeout 900 python bench.py --workload c5 --steps 100 2>/dev/null | tail -1 >> gpurun_out/bench_all.jsonl; echo "c5 rc=$?"
timeout 900 python bench.py --workload c5 --steps 100 --gate-first 2>/dev/null | tail -1 >> gpurun_out/bench_all.jsonl; echo "c5 gf rc=$?"
wc -l gpurun_out/bench_all.jsonl
