# round 2: new GPU tests (exchange, vstore churn, auto route), the torchrun 1-rank dry run of the
# multi-GPU path, and the default bench line
set -x
timeout 900 python -m pytest tests/test_gpu_auto.py tests/test_gpu_vstore.py tests/test_gpu_exchange.py tests/test_gpu_collective1.py -x -q 2>&1 | tail -15
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --steps 10 --warmup 3 --force-collective --no-cpu-baseline > gpurun_out/r02_dry_collective.json 2> gpurun_out/r02_dry_collective.err
echo "dry rc=$?"; tail -5 gpurun_out/r02_dry_collective.err
timeout 1200 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
echo "bench rc=$?"; tail -5 gpurun_out/r02_bench_default.err
