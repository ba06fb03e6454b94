#!/bin/bash
# usage: bash scripts/gpu_cmp.sh  -> gated/ungated C3 bench summaries
mkdir -p gpurun_out
python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-variant > gpurun_out/b_g.json 2> gpurun_out/b_g.err
python scripts/bench_summary.py gpurun_out/b_g.json gated
python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-variant --ungated > gpurun_out/b_u.json 2> gpurun_out/b_u.err
python scripts/bench_summary.py gpurun_out/b_u.json ungated
