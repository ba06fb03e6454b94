"""DRAM bytes of K2 vs query-tile count on C3's pool (ncu): does sharing a row split
across clusters re-read it from DRAM?"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import ams_gen
import paper_2508_10259_b200 as ams
dev = torch.device("cuda", 0)
cfg = ams_gen.CONFIGS["c3"]
nq = int(sys.argv[1])
pool = ams.Pool(cfg.d, cfg.J, cfg.M, nq, 16)
q, qj, lab = ams_gen.build_device_workload(cfg, dev, lambda e, j, n: pool.append(e, j, n), Q=nq)
for _ in range(3):
    pool.match(q, qj, 16, cfg.theta, cfg.gamma)
torch.cuda.synchronize()
print(nq, ams.ams_pool_last_plan(pool.handle))
