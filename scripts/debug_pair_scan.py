"""Debug: small-batch CTA-pair kernel on tiny pools (prints mismatches vs the oracle)."""
import numpy as np, torch, ams_gen, oracle, paper_2508_10259_b200 as ams
for M in (1, 37, 300, 700):
    for nq in (150, 256):
        cfg = ams_gen.small_variant("c3", M, nq)
        w = ams_gen.generate_host(cfg)
        with ams.Pool(cfg.d, cfg.J, cfg.M, 256, 16) as pool:
            pool.append(torch.from_numpy(w.emb).cuda(), torch.from_numpy(w.joints).cuda())
            for k in (1, 8):
                for gamma in (0.3, float("inf")):
                    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, k, cfg.theta, gamma)
                    i, s, h = (t.cpu().numpy() for t in pool.match(torch.from_numpy(w.q_emb).cuda(),
                               torch.from_numpy(w.q_joints).cuda(), k, cfg.theta, gamma))
                    plan = ams.ams_pool_last_plan(pool.handle)
                    bad = np.nonzero((i != orc.idx).any(1))[0]
                    print(M, nq, k, gamma, plan, "bad queries", bad.size, bad[:5],
                          i[bad[:2]].tolist() if bad.size else "", orc.idx[bad[:2]].tolist() if bad.size else "")
