#!/usr/bin/env python
"""Latency of one ams_match call vs batch size nq (diagnostic; GPU box).

    python scripts/nq_sweep.py [c5|c3] [--gate-first] [--policy P] [--k K] [--nq a,b,c]

Builds the config's pool with the ams_gen recipe, then times ams_match (CUDA events,
3 warm-ups, median of 10) for nq in 1..256 and prints ms, algorithmic GB/s and TF/s,
and the launch plan (splits, grid, kernel id) of each size.
"""
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import ams_gen  # noqa: E402
import paper_2508_10259_b200 as ams  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    gf = "--gate-first" in sys.argv
    arg = lambda f, d: type(d)(sys.argv[sys.argv.index(f) + 1]) if f in sys.argv else d  # noqa: E731
    policy, k = arg("--policy", 0), arg("--k", ams_gen.CONFIGS[name].k)
    cfg = ams_gen.CONFIGS[name]
    dev = torch.device("cuda", 0)
    nqs = [int(x) for x in arg("--nq", "1,2,4,8,16,32,64,96,128,129,160,192,224,256").split(",")]
    pool = ams.Pool(cfg.d, cfg.J, cfg.M, 256, max(k, cfg.k), dtype="bf16", device=0)
    ams.ams_pool_set_kernel_policy(pool.handle, policy)

    def append_fn(e, j, n):
        pool.append(e, j, n)

    q, qj, lab = ams_gen.build_device_workload(cfg, dev, append_fn, Q=256)
    torch.cuda.synchronize()
    oi = torch.empty(256, max(k, cfg.k), dtype=torch.int64, device=dev)
    os_ = torch.empty(256, max(k, cfg.k), dtype=torch.float32, device=dev)
    oh = torch.empty(256, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream()
    fn = ams.ams_match_gate_first if gf else ams.ams_match
    row_bytes = 2 * cfg.d + 4 * cfg.J + 4
    for gamma in (cfg.gamma, math.inf):
        for nq in nqs:
            for _ in range(3):
                fn(pool.handle, q[:nq], qj[:nq], nq, k, cfg.theta, gamma, oi, os_, oh, s)
            ts = []
            for _ in range(10):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                fn(pool.handle, q[:nq], qj[:nq], nq, k, cfg.theta, gamma, oi, os_, oh, s)
                b.record(s)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            ms = statistics.median(ts)
            plan = ams.ams_pool_last_plan(pool.handle)
            gbs = cfg.M * row_bytes / (ms * 1e-3) / 1e9
            tf = 2.0 * nq * cfg.M * cfg.d / (ms * 1e-3) / 1e12
            print(f"{name} policy={policy} k={k} gamma={gamma} nq={nq:4d} ms={ms:8.3f} min={min(ts):8.3f} max={max(ts):8.3f} "
                  f"GB/s={gbs:7.0f} TF/s={tf:7.1f} plan={plan}", flush=True)
    pool.close()


if __name__ == "__main__":
    main()
