"""Edge cases and error behaviour of the C ABI on the GPU."""
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


def dev():
    return torch.device("cuda", 0)


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


def outs(nq, k):
    return (torch.empty(nq, k, dtype=torch.int64, device=dev()), torch.empty(nq, k, dtype=torch.float32, device=dev()),
            torch.empty(nq, dtype=torch.uint8, device=dev()))


def test_argument_errors(ams):
    w = ams_gen.generate_host(ams_gen.small_variant("c2", 500, 8))
    with ams.Pool(768, 7, 1000, 8, 10) as pool:
        pool.append(T(w.emb), T(w.joints))
        q, qj = T(w.q_emb), T(w.q_joints)
        oi, os_, oh = outs(8, 10)
        bad = [dict(nq=0), dict(nq=9), dict(k=0), dict(k=11), dict(theta=float("nan")),
               dict(gamma=-0.1), dict(gamma=float("nan"))]
        for b in bad:
            a = dict(nq=8, k=10, theta=0.5, gamma=0.3)
            a.update(b)
            with pytest.raises(ams.AmsError) as e:
                ams.ams_match(pool.handle, q, qj, a["nq"], a["k"], a["theta"], a["gamma"], oi, os_, oh)
            assert e.value.status == 1, b
        with pytest.raises(ams.AmsError) as e:
            ams.ams_match(pool.handle, q, qj, 8, 10, 0.5, 0.3, None, os_, oh)
        assert e.value.status == 1
        # the pool is still usable after argument errors
        pool.match(q, qj, 10, 0.5, 0.3)
        torch.cuda.synchronize()


def test_capacity_error_is_all_or_nothing(ams):
    w = ams_gen.generate_host(ams_gen.small_variant("c2", 700, 8))
    with ams.Pool(768, 7, 600, 8, 10) as pool:
        assert pool.append(T(w.emb[:500]), T(w.joints[:500])) == 0
        with pytest.raises(ams.AmsError) as e:
            pool.append(T(w.emb[500:700]), T(w.joints[500:700]))
        assert e.value.status == 2
        assert pool.size == 500
        assert pool.append(T(w.emb[500:600]), T(w.joints[500:600])) == 500
        assert pool.size == 600
        oi, os_, oh = pool.match(T(w.q_emb), T(w.q_joints), 10, 0.9, INF)
        orc = oracle.match(w.emb[:600], w.joints[:600], w.q_emb, w.q_joints, 10, 0.9, INF)
        check_bf16(oi.cpu().numpy(), os_.cpu().numpy(), oh.cpu().numpy(), orc, 0.9)


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_empty_pool_and_k_larger_than_pool(ams, dtype):
    cfg = ams_gen.small_variant("c2", 20, 5) if dtype == "bf16" else ams_gen.CONFIGS["c1"]
    w = ams_gen.generate_host(cfg)
    d = w.emb.shape[1]
    with ams.Pool(d, cfg.J, 100, 64, 32, dtype=dtype) as pool:
        oi, os_, oh = pool.match(T(w.q_emb[:5]), T(w.q_joints[:5]), 7, -INF, INF)
        torch.cuda.synchronize()
        assert (oi.cpu().numpy() == -1).all() and (oh.cpu().numpy() == 0).all()
        assert np.isneginf(os_.cpu().numpy()).all()
        pool.append(T(w.emb[:20]), T(w.joints[:20]))
        oi, os_, oh = pool.match(T(w.q_emb[:5]), T(w.q_joints[:5]), 32, 0.5, INF)
        torch.cuda.synchronize()
        orc = oracle.match(w.emb[:20], w.joints[:20], w.q_emb[:5], w.q_joints[:5], 32, 0.5, INF)
        if dtype == "fp32":
            check_exact(oi.cpu().numpy(), os_.cpu().numpy(), oh.cpu().numpy(), orc)
        else:
            check_bf16(oi.cpu().numpy(), os_.cpu().numpy(), oh.cpu().numpy(), orc, 0.5)
        assert (oi.cpu().numpy()[:, 20:] == -1).all()


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_streaming_appends_interleaved_with_matches(ams, dtype):
    """C5-style record-and-replay: appends of varying sizes (host and device sources)
    interleaved with matches; each match sees exactly the rows appended before it."""
    cfg = ams_gen.small_variant("c5", 6000, 40) if dtype == "bf16" else ams_gen.small_variant("c1", 3000, 40)
    w = ams_gen.generate_host(cfg)
    rng = np.random.Generator(np.random.PCG64(9))
    with ams.Pool(w.emb.shape[1], cfg.J, cfg.M, cfg.Q, cfg.k, dtype=dtype, shard_block=256) as pool:
        n = 0
        step = 0
        while n < cfg.M:
            m = int(min(cfg.M - n, rng.integers(1, 900)))
            src_e, src_j = w.emb[n:n + m], w.joints[n:n + m]
            if step % 2:
                first = pool.append(np.ascontiguousarray(src_e), np.ascontiguousarray(src_j), m)
            else:
                first = pool.append(T(src_e), T(src_j), m)
            assert first == n
            n += m
            step += 1
            if step % 3 == 0 or n == cfg.M:
                nq = int(rng.integers(1, cfg.Q + 1))
                gamma = cfg.gamma if step % 2 else INF
                oi, os_, oh = pool.match(T(w.q_emb[:nq]), T(w.q_joints[:nq]), cfg.k, cfg.theta, gamma)
                torch.cuda.synchronize()
                orc = oracle.match(w.emb[:n], w.joints[:n], w.q_emb[:nq], w.q_joints[:nq], cfg.k, cfg.theta, gamma)
                g = (oi.cpu().numpy(), os_.cpu().numpy(), oh.cpu().numpy())
                if dtype == "fp32":
                    check_exact(*g, orc)
                else:
                    check_bf16(*g, orc, cfg.theta)


def test_zero_norm_rows_and_infinite_thresholds(ams):
    cfg = ams_gen.small_variant("c3", 2000, 50)
    w = ams_gen.generate_host(cfg)
    emb = w.emb.copy()
    emb[::97] = 0                      # zero rows -> score exactly 0 (R8)
    q = w.q_emb.copy()
    q[3] = 0                           # zero query -> all scores 0, ranked by index
    for theta in (-INF, INF, 0.0):
        orc = oracle.match(emb, w.joints, q, w.q_joints, cfg.k, theta, INF)
        with ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k) as pool:
            pool.append(T(emb), T(w.joints))
            oi, os_, oh = pool.match(T(q), T(w.q_joints), cfg.k, theta, INF)
            torch.cuda.synchronize()
            g = (oi.cpu().numpy(), os_.cpu().numpy(), oh.cpu().numpy())
        check_bf16(*g, orc, theta)
        assert g[0][3].tolist() == list(range(cfg.k)) and (g[1][3] == 0).all()


def test_max_queries_exactly(ams):
    cfg = ams_gen.small_variant("c2", 8000, 1000)
    w = ams_gen.generate_host(cfg)
    with ams.Pool(cfg.d, cfg.J, cfg.M, 1000, cfg.k) as pool:
        pool.append(T(w.emb), T(w.joints))
        oi, os_, oh = pool.match(T(w.q_emb), T(w.q_joints), cfg.k, cfg.theta, cfg.gamma)
        torch.cuda.synchronize()
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, cfg.gamma, mode="B")
    check_bf16(oi.cpu().numpy(), os_.cpu().numpy(), oh.cpu().numpy(), orc, cfg.theta)
