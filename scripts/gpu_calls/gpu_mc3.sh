mkdir -p gpurun_out
python - <<'PY'
import torch, numpy as np, paper_2508_10259_b200 as ams, ams_gen
cfg = ams_gen.small_variant("c3", 300000, 16384)
pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k)
e = torch.zeros(cfg.M, cfg.d, dtype=torch.bfloat16, device="cuda"); j = torch.zeros(cfg.M, cfg.J, device="cuda")
pool.append(e, j)
q = torch.zeros(cfg.Q, cfg.d, dtype=torch.bfloat16, device="cuda"); qj = torch.zeros(cfg.Q, cfg.J, device="cuda")
for pol in (0, 2):
    ams.ams_pool_set_kernel_policy(pool.handle, pol); pool.match(q, qj, 16, 0.9, 0.3); torch.cuda.synchronize()
    print("policy", pol, ams.ams_pool_last_plan(pool.handle))
PY
python scripts/diag_power.py multicast 2>&1 | grep label
AMS_POLICY=2 python scripts/diag_power.py pair 2>&1 | grep label
