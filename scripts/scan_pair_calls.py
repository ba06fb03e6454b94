"""C3's pool (1M x 1024), 200 queries, k = 8: the small-batch kernel on CTA pairs (for ncu)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import ams_gen
import paper_2508_10259_b200 as ams
dev = torch.device("cuda", 0)
cfg = ams_gen.CONFIGS["c3"]
pool = ams.Pool(cfg.d, cfg.J, cfg.M, 256, 8)
q, qj, lab = ams_gen.build_device_workload(cfg, dev, lambda e, j, n: pool.append(e, j, n), Q=256)
for _ in range(4):
    pool.match(q[:200], qj[:200], 8, cfg.theta, cfg.gamma)
torch.cuda.synchronize()
print(ams.ams_pool_last_plan(pool.handle))
if os.environ.get("TIME"):
    for gamma in (cfg.gamma, float("inf")):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            pool.match(q[:200], qj[:200], 8, cfg.theta, gamma)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print("gamma", gamma, "ms/call", round(ms, 4), "GB/s", round(cfg.M * (2 * cfg.d + 4 * cfg.J + 4) / ms / 1e6))
