"""Short-burst comparison (not power capped): C3 gated kernel time with variants."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch, ams_gen
import paper_2508_10259_b200 as ams
torch.cuda.set_device(0); dev = torch.device("cuda", 0)
cfg = ams_gen.CONFIGS["c3"]
pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k)
q, qj, lab = ams_gen.build_device_workload(cfg, dev, lambda e, j, n: pool.append(e, j, n))
out = pool.match(q, qj, cfg.k, cfg.theta, cfg.gamma)
for gamma in (cfg.gamma, float("inf")):
    ts = []
    for rep in range(6):
        time.sleep(0.5)
        ams.ams_pool_set_profiling(pool.handle, True)
        pool.match(q, qj, cfg.k, cfg.theta, gamma, out=out)
        torch.cuda.synchronize()
        ms, n = ams.ams_pool_read_profile(pool.handle)
        ts.append(ms)
    print(json.dumps({"lib": os.environ.get("AMS_LIBRARY", "product"), "gamma": gamma, "ms": sorted(ts)[:3]}))
