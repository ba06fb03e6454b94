"""Exact-path activity of the dense epilogue (diag build with AMS_DIAG_COUNT):
chunks, firing 8-column sub-chunks, inserts, per config and gate.
Run: AMS_LIBRARY=$PWD/diag_lib/libams_diag_ams_diag_count.so python scripts/diag_count.py"""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
import ams_gen
import paper_2508_10259_b200 as ams
lib = ctypes.CDLL(ams.LIB_PATH)
buf = (ctypes.c_ulonglong * 4)()
dev = torch.device("cuda", 0)
cfg = ams_gen.CONFIGS["c3"]
pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k)
q, qj, lab = ams_gen.build_device_workload(cfg, dev, lambda e, j, n: pool.append(e, j, n))
print("pool built", flush=True)
for nq in (1, 64, 16384):
    for gamma in (cfg.gamma, float("inf")):
        pool.match(q[:nq], qj[:nq], cfg.k, cfg.theta, gamma)
        torch.cuda.synchronize()
        lib.ams_diag_counts(buf, 1)
        pool.match(q[:nq], qj[:nq], cfg.k, cfg.theta, gamma)
        torch.cuda.synchronize()
        lib.ams_diag_counts(buf, 1)
        ch, fire, ins = buf[0], buf[1], buf[2]
        print(f"nq={nq} gamma={gamma} chunks={ch} firing_subchunks={fire} ({fire / max(ch, 1) / 4:.4f} of sub-chunks) "
              f"inserts={ins} ({ins / nq:.1f} per query) plan={ams.ams_pool_last_plan(pool.handle)}", flush=True)
