"""configs[0] (fp32 exact) calls, gated and ungated, for an ncu launch list."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, ams_gen, paper_2508_10259_b200 as ams
cfg = ams_gen.CONFIGS["c1"]
w = ams_gen.generate_host(cfg)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k, dtype="fp32")
pool.append(T(w.emb), T(w.joints))
q, qj = T(w.q_emb), T(w.q_joints)
for gamma in (cfg.gamma, float("inf")):
    for _ in range(3):
        pool.match(q, qj, cfg.k, cfg.theta, gamma)
torch.cuda.synchronize()
print(ams.ams_pool_last_plan(pool.handle))
