"""Latency of one configs[0] (fp32 exact) ams_match call, gated and ungated, k = 5 and 32."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, ams_gen, paper_2508_10259_b200 as ams
cfg = ams_gen.CONFIGS["c1"]; w = ams_gen.generate_host(cfg)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, 64, dtype="fp32"); pool.append(T(w.emb), T(w.joints))
q, qj = T(w.q_emb), T(w.q_joints)
for g in (cfg.gamma, float("inf")):
    for k in (5, 32):
        for _ in range(5): pool.match(q, qj, k, cfg.theta, g)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200): pool.match(q, qj, k, cfg.theta, g)
        e1.record(); torch.cuda.synchronize()
        print("gamma", g, "k", k, "us/call", round(e0.elapsed_time(e1) / 200 * 1e3, 1))
