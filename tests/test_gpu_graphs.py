"""ams_match inside CUDA graphs: the call is stream-ordered and host-decided (plan from the
pool size, no host synchronisation), so a captured call replays with new query contents
written into the same device buffers.  Checked against the oracle on every replay for
the fp32 exact kernel (configs[0], bit-exact), the small-batch tcgen05 kernel and the
CTA-pair kernel; a graph must be re-captured after appends (the plan is frozen)."""
import numpy as np
import pytest

import ams_gen
import oracle
from tests.parity import check_bf16, check_exact

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
INF = float("inf")


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


def dev_t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.device("cuda", 0))


@pytest.mark.parametrize("name,M,Q", [("c1", 1024, 64), ("c3", 3001, 64), ("c2", 5000, 300)])
@pytest.mark.parametrize("gated", [True, False])
def test_match_replays_in_cuda_graph(ams, name, M, Q, gated):
    cfg = ams_gen.CONFIGS["c1"] if name == "c1" else ams_gen.small_variant(name, M, Q)
    w = ams_gen.generate_host(cfg)
    w2 = ams_gen.generate_host(ams_gen.small_variant(name, cfg.M, cfg.Q, seed_offset=200)
                               if name != "c1" else ams_gen.small_variant("c1", cfg.M, cfg.Q, seed_offset=200))
    gamma = cfg.gamma if gated else INF
    dt = "fp32" if cfg.dtype == "fp32" else "bf16"
    with ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k, dtype=dt) as pool:
        pool.append(dev_t(w.emb), dev_t(w.joints))
        q, qj = dev_t(w.q_emb), dev_t(w.q_joints)
        out = (torch.empty(cfg.Q, cfg.k, dtype=torch.int64, device="cuda"),
               torch.empty(cfg.Q, cfg.k, dtype=torch.float32, device="cuda"),
               torch.empty(cfg.Q, dtype=torch.uint8, device="cuda"))
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):   # warm-up outside capture (function attributes, lazy state)
            pool.match(q, qj, cfg.k, cfg.theta, gamma, out=out, stream=s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            pool.match(q, qj, cfg.k, cfg.theta, gamma, out=out, stream=s)
        for src in (w, w2, w):   # new query contents in the captured buffers, then replay
            q.copy_(dev_t(src.q_emb))
            qj.copy_(dev_t(src.q_joints))
            for t in out:
                t.fill_(0)
            g.replay()
            torch.cuda.synchronize()
            orc = oracle.match(w.emb, w.joints, src.q_emb, src.q_joints, cfg.k, cfg.theta, gamma)
            got = tuple(t.cpu().numpy() for t in out)
            if dt == "fp32":
                check_exact(*got, orc)
            else:
                check_bf16(*got, orc, cfg.theta)
