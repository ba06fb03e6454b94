"""Route selection by estimated pass-rate (ams_match_auto, SURVEY.md 8(f) f3 "select by
measured pass-rate"): both routes against the oracle, and the route the cost model must
pick in the regimes it separates."""
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


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("name,M,Q,gamma,route", [
    ("c3", 120011, 300, 0.3, "gate_first"),   # R14 gate: ~0-1 eligible rows per query
    ("c3", 120011, 64, 0.3, "gate_first"),
    ("c2", 40000, 257, 3.5, "dense"),         # J = 7, gamma 3.5: ~8 % of rows eligible -> buckets overflow
    ("c2", 40000, 64, INF, "dense"),          # ungated: always dense
])
def test_auto_route_and_parity(ams, name, M, Q, gamma, route):
    cfg = ams_gen.small_variant(name, M, Q)
    w = ams_gen.generate_host(cfg)
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma, mode="B")
    with ams.Pool(cfg.d, cfg.J, M, Q, cfg.k) as pool:
        pool.append(T(w.emb), T(w.joints))
        for rep in range(3):   # first call estimates synchronously, later ones reuse the cache
            out = pool.match(T(w.q_emb), T(w.q_joints), cfg.k, cfg.theta, gamma, gate_first="auto")
            torch.cuda.synchronize()
            r = ams.ams_pool_last_route(pool.handle)
            assert r["route"] == route, (rep, r)
            assert (ams.ams_pool_last_plan(pool.handle)["kernel_id"] == 3) == (route == "gate_first")
            check_bf16(*[t.cpu().numpy() for t in out], orc, cfg.theta)
        if np.isfinite(gamma):
            nelig = orc.nelig.mean()
            est = r["est_eligible_per_query"]
            # the sampled estimate is within a loose factor of the exact mean (or both tiny)
            assert (est <= 4 * nelig + 2) and (est >= nelig / 4 - 2), (est, nelig)


def test_auto_estimate_refreshes_on_gamma_change(ams):
    cfg = ams_gen.small_variant("c2", 120011, 128)
    w = ams_gen.generate_host(cfg)
    with ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k) as pool:
        pool.append(T(w.emb), T(w.joints))
        routes = []
        for gamma in (0.3, 3.5, 0.3):
            pool.match(T(w.q_emb), T(w.q_joints), cfg.k, cfg.theta, gamma, gate_first="auto")
            torch.cuda.synchronize()
            routes.append(ams.ams_pool_last_route(pool.handle)["route"])
        assert routes == ["gate_first", "dense", "gate_first"]


def test_auto_many_calls_async_refresh(ams):
    """> 64 calls: the asynchronous refresh path runs and keeps choosing correctly."""
    cfg = ams_gen.small_variant("c3", 120011, 96)
    w = ams_gen.generate_host(cfg)
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, cfg.gamma, mode="B")
    with ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k) as pool:
        pool.append(T(w.emb), T(w.joints))
        q, qj = T(w.q_emb), T(w.q_joints)
        for _ in range(140):
            out = pool.match(q, qj, cfg.k, cfg.theta, cfg.gamma, gate_first="auto")
        torch.cuda.synchronize()
        assert ams.ams_pool_last_route(pool.handle)["route"] == "gate_first"
        check_bf16(*[t.cpu().numpy() for t in out], orc, cfg.theta)


def test_auto_fp32_is_exact(ams):
    cfg = ams_gen.CONFIGS["c1"]
    w = ams_gen.generate_host(cfg)
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, cfg.gamma)
    with ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k, dtype="fp32") as pool:
        pool.append(T(w.emb), T(w.joints))
        out = pool.match(T(w.q_emb), T(w.q_joints), cfg.k, cfg.theta, cfg.gamma, gate_first="auto")
        torch.cuda.synchronize()
        assert ams.ams_pool_last_route(pool.handle)["route"] == "dense"
        check_exact(*[t.cpu().numpy() for t in out], orc)
