# round 2 end-of-round style check: full GPU suite, smoke, the default bench line, the
# torchrun 1-rank dry run of the multi-GPU path
set -x
sha256sum paper_2508_10259_b200/libams.so
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/r02_bench_final2.json 2> gpurun_out/r02_bench_final2.err; echo "bench rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --steps 10 --warmup 3 --force-collective --no-cpu-baseline > gpurun_out/r02_dry_collective2.json 2> gpurun_out/r02_dry_collective2.err
echo "dry rc=$?"
