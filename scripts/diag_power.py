"""Power/clock diagnostic: full kernel vs the MMA+TMA pipeline alone (epilogue compiled
out, build/diag/libams_diag.so) vs cuBLAS, each for ~3 s under nvidia-smi sampling.
Run: [AMS_LIBRARY=...] [AMS_POLICY=<ams_pool_set_kernel_policy mask>] python scripts/diag_power.py <label>"""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench
import ams_gen
label = sys.argv[1]
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
def timed(fn, secs=3.0):
    fn(); torch.cuda.synchronize()
    clk = bench.ClockSampler(0); clk.start(); time.sleep(0.2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0; t_end = time.time() + secs; e0.record()
    while time.time() < t_end:
        fn(); n += 1
        if n % 4 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, clk.stop()
if label == "cublas":
    A = torch.randn(16384, 1024, device=dev, dtype=torch.bfloat16)
    B = torch.randn(1024, 65536, device=dev, dtype=torch.bfloat16)
    C = torch.empty(16384, 65536, device=dev, dtype=torch.bfloat16)
    ms, clk = timed(lambda: torch.matmul(A, B, out=C))
    print(json.dumps({"label": label, "ms": ms, "tflops": 2*16384*65536*1024/ms/1e9, "clocks": clk}))
    sys.exit(0)
import paper_2508_10259_b200 as ams
print("lib", ams.LIB_PATH)
cfg = ams_gen.CONFIGS["c3"]
pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k)
ams.ams_pool_set_kernel_policy(pool.handle, int(os.environ.get("AMS_POLICY", "0")))
q, qj, lab = ams_gen.build_device_workload(cfg, dev, lambda e, j, n: pool.append(e, j, n))
out = pool.match(q, qj, cfg.k, cfg.theta, cfg.gamma)
for gamma in (cfg.gamma, float("inf")):
    ms, clk = timed(lambda: pool.match(q, qj, cfg.k, cfg.theta, gamma, out=out))
    print(json.dumps({"label": label, "gamma": gamma, "ms": ms, "tflops": 2*cfg.Q*cfg.M*cfg.d/ms/1e9, "clocks": clk}))
