#!/usr/bin/env python
"""A few identical ams_match calls on a config's pool, for ncu captures of one kernel.

    python scripts/one_call.py c3 --nq 200 --k 8 [--policy P] [--gamma G] [--calls N] [--gate-first | --auto] [--timeline]

Builds the pool with the ams_gen recipe (not timed), then issues N calls (default 5);
prints the median CUDA-event time per call and the plan.  ncu: -k regex:match_scan
--launch-skip 3 -c 1 captures the 4th call's kernel.  --timeline then prints the kernels of
three back-to-back calls with their in-stream durations and the idle gaps between them.
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
    name = sys.argv[1]
    arg = lambda f, d: type(d)(sys.argv[sys.argv.index(f) + 1]) if f in sys.argv else d  # noqa: E731
    cfg = ams_gen.CONFIGS[name]
    nq, k, policy, calls = arg("--nq", 64), arg("--k", cfg.k), arg("--policy", 0), arg("--calls", 5)
    gamma = arg("--gamma", cfg.gamma)
    dev = torch.device("cuda", 0)
    pool = ams.Pool(cfg.d, cfg.J, cfg.M, max(nq, 1), max(k, 1), dtype="bf16", device=0)
    ams.ams_pool_set_kernel_policy(pool.handle, policy)
    if cfg.dtype == "fp32":   # configs[0]: the host recipe (no mixture components)
        w = ams_gen.generate_host(cfg)
        pool.close()
        pool = ams.Pool(cfg.d, cfg.J, cfg.M, max(nq, 1), max(k, 1), dtype="fp32", device=0)
        ams.ams_pool_set_kernel_policy(pool.handle, policy)
        pool.append(torch.from_numpy(w.emb).to(dev), torch.from_numpy(w.joints).to(dev))
        reps = (nq + cfg.Q - 1) // cfg.Q
        q = torch.from_numpy(w.q_emb).to(dev).repeat(reps, 1)
        qj = torch.from_numpy(w.q_joints).to(dev).repeat(reps, 1)
    else:
        q, qj, _ = ams_gen.build_device_workload(cfg, dev, lambda e, j, n: pool.append(e, j, n), Q=max(nq, 64))
    q, qj = q[:nq].contiguous(), qj[:nq].contiguous()
    out = (torch.empty(nq, k, dtype=torch.int64, device=dev), torch.empty(nq, k, dtype=torch.float32, device=dev),
           torch.empty(nq, dtype=torch.uint8, device=dev))
    fn = ams.ams_match_gate_first if "--gate-first" in sys.argv else ams.ams_match
    if "--auto" in sys.argv:   # the routed entry point (cost model; may run the gate estimate)
        fn = ams.ams_match_auto
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(calls):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn(pool.handle, q, qj, nq, k, cfg.theta, gamma, *out, s)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    row_bytes = 2 * cfg.d + 4 * cfg.J + 4
    ms = statistics.median(ts)
    print(f"{name} nq={nq} k={k} gamma={gamma} policy={policy} ms={ms:.4f} GB/s={cfg.M * row_bytes / ms / 1e6:.0f} "
          f"plan={ams.ams_pool_last_plan(pool.handle)}", flush=True)
    if "--timeline" in sys.argv:
        # in-stream kernel durations and the gaps between them (CUPTI via torch.profiler;
        # natural clocks and warm L2, unlike a serialised ncu launch list)
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(3):
                fn(pool.handle, q, qj, nq, k, cfg.theta, gamma, *out, s)
            torch.cuda.synchronize()
        evs = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
        prev = None
        for e in evs:
            gap = "" if prev is None else f" gap={e.time_range.start - prev:8.2f}"
            print(f"    {e.name.split('(')[0][:60]:60s} dur={e.time_range.elapsed_us():8.2f} us{gap}", flush=True)
            prev = e.time_range.end


if __name__ == "__main__":
    main()
