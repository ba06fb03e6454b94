import itertools, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
os.environ["AMS_LOG"] = "1"
import ams_gen, oracle
import paper_2508_10259_b200 as ams
rows = np.array(list(itertools.product([-1.0, 1.0], repeat=4)), np.float32)
rng = np.random.Generator(np.random.PCG64(11))
joints = rng.integers(-2, 3, (16, 2)).astype(np.float32)
qj = np.array([[0, 0], [1, -1], [2, 2], [-2, 1]] * 4, np.float32)
e = np.zeros((16, 64), np.float32); e[:, :4] = rows
e = ams_gen.f32_to_bf16_bits(e)
dev = torch.device("cuda", 0)
for gamma in (0.0, 1.0, 2.0, float("inf")):
    for k in (1, 3, 5, 16, 17):
        pool = ams.Pool(64, 2, 16, 16, 32)
        pool.append(torch.from_numpy(e).to(dev), torch.from_numpy(joints).to(dev))
        try:
            out = pool.match(torch.from_numpy(e).to(dev), torch.from_numpy(qj).to(dev), k, 0.5, gamma)
            torch.cuda.synchronize()
            print("ok", gamma, k, ams.ams_pool_last_plan(pool.handle), flush=True)
        except Exception as ex:
            print("FAIL", gamma, k, ex, flush=True)
            err = torch.cuda.synchronize() if False else None
            sys.exit(1)
        pool.close()
