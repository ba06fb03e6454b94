"""Small-batch ungated/gated calls on the C3 pool (for an ncu launch list)."""
import math, os, sys
sys.path.insert(0, os.getcwd())
import torch
import ams_gen
import paper_2508_10259_b200 as ams
dev = torch.device("cuda", 0)
cfg = ams_gen.CONFIGS["c3"]
pool = ams.Pool(cfg.d, cfg.J, cfg.M, 256, cfg.k)
q, qj, lab = ams_gen.build_device_workload(cfg, dev, lambda e, j, n: pool.append(e, j, n), Q=256)
for nq in (1, 64):
    for gamma in (cfg.gamma, math.inf):
        for _ in range(3):
            pool.match(q[:nq], qj[:nq], cfg.k, cfg.theta, gamma)
        torch.cuda.synchronize()
print("done")
