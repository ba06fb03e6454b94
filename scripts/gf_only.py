"""Gate-first timing alone (no preceding dense load): C3 pool, 16384 / 64 / 1 queries."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch, ams_gen
import paper_2508_10259_b200 as ams
torch.cuda.set_device(0); dev = torch.device("cuda", 0)
cfg = ams_gen.CONFIGS["c3"]
pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k)
q, qj, lab = ams_gen.build_device_workload(cfg, dev, lambda e, j, n: pool.append(e, j, n))
time.sleep(2)
for nq in (cfg.Q, 64, 1):
    qq, qqj = q[:nq].contiguous(), qj[:nq].contiguous()
    out = pool.match(qq, qqj, cfg.k, cfg.theta, cfg.gamma, gate_first=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); pool.match(qq, qqj, cfg.k, cfg.theta, cfg.gamma, out=out, gate_first=True); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"nq": nq, "ms_median": ts[5], "ms_min": ts[0], "q_per_s": nq / ts[5] * 1e3}))
