"""Hash throughput (ams_hash_actions) on 64 x 16 MB blobs, 1M 57-byte actions, and a mix."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2508_10259_b200 as ams
torch.cuda.set_device(0)
for label, lens in [("blobs_16MB", np.full(64, 16 << 20)), ("actions_57B", np.full(1 << 20, 57)),
                    ("mixed", np.concatenate([np.full(32, 16 << 20), np.full(1 << 19, 57)]))]:
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    data = torch.randint(0, 256, (int(offs[-1]),), dtype=torch.uint8, device="cuda")
    n = len(lens)
    h = ams.ams_hasher_create(0, n, int(offs[-1]), 4096)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    for _ in range(3): ams.ams_hash_actions(h, data, offs, n, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    t0 = time.perf_counter()
    for _ in range(reps): ams.ams_hash_actions(h, data, offs, n, out)
    host_ms = (time.perf_counter() - t0) * 1e3 / reps   # enqueue cost per call (host bookkeeping)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"case": label, "bytes": int(offs[-1]), "inputs": n, "ms": ms, "GBps": offs[-1] / ms / 1e6, "host_enqueue_ms": host_ms,
                      **ams.ams_hasher_last_stats(h)}))
    ams.ams_hasher_destroy(h)
