"""Gate-first vs dense timing on C3 (16384 q) and a 64-query batch."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, ams_gen
import paper_2508_10259_b200 as ams
torch.cuda.set_device(0); dev = torch.device("cuda", 0)
cfg = ams_gen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k)
q, qj, lab = ams_gen.build_device_workload(cfg, dev, lambda e, j, n: pool.append(e, j, n))
for nq in (cfg.Q, 64, 1):
    for gf in (False, True):
        qq, qqj = q[:nq].contiguous(), qj[:nq].contiguous()
        out = pool.match(qq, qqj, cfg.k, cfg.theta, cfg.gamma, gate_first=gf)
        for _ in range(3): pool.match(qq, qqj, cfg.k, cfg.theta, cfg.gamma, out=out, gate_first=gf)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps): pool.match(qq, qqj, cfg.k, cfg.theta, cfg.gamma, out=out, gate_first=gf)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"cfg": cfg.name, "nq": nq, "gate_first": gf, "ms_per_call": ms, "q_per_s": nq / ms * 1e3}))
