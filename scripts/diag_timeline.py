"""Diagnostic: per-unit timeline of match_tc_kernel (diag build AMS_DIAG_TIMELINE).

Usage (on the GPU box):
  AMS_LIBRARY=$PWD/diag_lib/libams_diag_ams_diag_timeline.so python scripts/diag_timeline.py c4 out.npz
Runs 3 warm-up matches + 1 recorded match, saves (start_ns, end_ns, cluster, smid) per
unit plus the plan, to study how far apart in time the units sharing a row split run.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import ams_gen  # noqa: E402
import paper_2508_10259_b200 as ams  # noqa: E402


def main():
    name, out = sys.argv[1], sys.argv[2]
    cfg = ams_gen.CONFIGS[name]
    dev = torch.device("cuda", 0)
    pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k)
    q, qj, _ = ams_gen.build_device_workload(cfg, dev, lambda e, j, n: pool.append(e, j, n),
                                             chunk_needed=lambda lo, hi: True)
    torch.cuda.synchronize()
    oi = torch.empty(cfg.Q, cfg.k, dtype=torch.int64, device=dev)
    os_ = torch.empty(cfg.Q, cfg.k, dtype=torch.float32, device=dev)
    oh = torch.empty(cfg.Q, dtype=torch.uint8, device=dev)
    for _ in range(4):
        ams.ams_match(pool.handle, q, qj, cfg.Q, cfg.k, cfg.theta, cfg.gamma, oi, os_, oh)
    torch.cuda.synchronize()
    plan = ams.ams_pool_last_plan(pool.handle)
    S, grid = plan["splits"], plan["grid"]
    n_units = ((cfg.Q + 255) // 256) * S
    buf = (ctypes.c_ulonglong * (n_units * 3))()
    rc = ams.lib.ams_diag_timeline(buf, n_units)
    assert rc == 0, rc
    a = np.frombuffer(buf, dtype=np.uint64).reshape(n_units, 3)
    np.savez(out, start=a[:, 0], end=a[:, 1], cid=(a[:, 2] & 0xffffffff), smid=(a[:, 2] >> 32), S=S, grid=grid,
             n_qt=(cfg.Q + 255) // 256)
    t0 = a[:, 0].min()
    st = (a[:, 0] - t0) / 1e6
    en = (a[:, 1] - t0) / 1e6
    n_qt = (cfg.Q + 255) // 256
    spread = []
    for sp in range(S):
        u = np.arange(sp * n_qt, (sp + 1) * n_qt)
        spread.append(st[u].max() - st[u].min())
    dur = en - st
    print(f"{name}: S={S} grid={grid} units={n_units} total={en.max():.1f} ms; unit dur mean {dur.mean():.2f} "
          f"min {dur.min():.2f} max {dur.max():.2f} ms; start spread per split: median {np.median(spread):.2f} "
          f"max {np.max(spread):.2f} ms")


if __name__ == "__main__":
    main()
