"""Latency of one ams_match call issued directly vs replayed from a CUDA graph
(launch-bound small cases: configs[0] fp32 exact, and a 64-query bf16 call on a 20K pool)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import ams_gen
import paper_2508_10259_b200 as ams

def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()

for name, cfg in (("c1", ams_gen.CONFIGS["c1"]), ("c3-20k-64q", ams_gen.small_variant("c3", 20000, 64))):
    w = ams_gen.generate_host(cfg)
    dt = "fp32" if cfg.dtype == "fp32" else "bf16"
    pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k, dtype=dt)
    pool.append(T(w.emb), T(w.joints))
    q, qj = T(w.q_emb), T(w.q_joints)
    out = (torch.empty(cfg.Q, cfg.k, dtype=torch.int64, device="cuda"),
           torch.empty(cfg.Q, cfg.k, dtype=torch.float32, device="cuda"),
           torch.empty(cfg.Q, dtype=torch.uint8, device="cuda"))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(5):
            pool.match(q, qj, cfg.k, cfg.theta, cfg.gamma, out=out, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        pool.match(q, qj, cfg.k, cfg.theta, cfg.gamma, out=out, stream=s)
    n = 200
    for label, fn in (("direct", lambda: pool.match(q, qj, cfg.k, cfg.theta, cfg.gamma, out=out, stream=s)),
                      ("graph", g.replay)):
        with torch.cuda.stream(s):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(n):
                fn()
            e1.record(s)
        s.synchronize()
        print(name, label, "us/call", round(e0.elapsed_time(e1) / n * 1e3, 1))
    pool.close()
