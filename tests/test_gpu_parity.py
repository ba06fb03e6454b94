"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Every test is @pytest.mark.gpu.  Inputs come from ams_gen (seeded); expected values
come only from oracle/ (never from the CUDA path).
"""
import itertools
import json
import os

import numpy as np
import pytest

import ams_gen
import oracle
from tests.parity import check_bf16, check_exact

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
INF = float("inf")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


def dev():
    return torch.device("cuda", 0)


def to_dev(a):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to(dev())


def run_gpu(ams, w_emb, w_joints, q, qj, k, theta, gamma, dtype, max_k=None, host_inputs=False, pool=None):
    """Create a pool, append, match; returns numpy (idx, score, hit)."""
    M, d = w_emb.shape
    J = w_joints.shape[1]
    nq = q.shape[0]
    own = pool is None
    if own:
        pool = ams.Pool(d, J, max(M, 1), max(nq, 1), max_k or k, dtype=dtype)
        if M:
            if host_inputs:
                pool.append(np.ascontiguousarray(w_emb), np.ascontiguousarray(w_joints, np.float32), M)
            else:
                pool.append(to_dev(w_emb), to_dev(w_joints.astype(np.float32)), M)
    if host_inputs:
        out = pool.match(np.ascontiguousarray(q), np.ascontiguousarray(qj, np.float32), k, theta, gamma)
    else:
        out = pool.match(to_dev(q), to_dev(qj.astype(np.float32)), k, theta, gamma)
    torch.cuda.synchronize()
    res = tuple(t.cpu().numpy() for t in out)
    if own:
        pool.close()
    return res


def pad_d(x, d=64):
    out = np.zeros((x.shape[0], d), x.dtype)
    out[:, : x.shape[1]] = x
    return out


# ---------------------------------------------------------------------------- C1 exact
@pytest.mark.parametrize("gamma", [0.3, INF])
@pytest.mark.parametrize("host_inputs", [False, True])
def test_c1_fp32_bit_exact(ams, gamma, host_inputs):
    cfg = ams_gen.CONFIGS["c1"]
    w = ams_gen.generate_host(cfg)
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma)
    g = run_gpu(ams, w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma, "fp32",
                host_inputs=host_inputs)
    check_exact(*g, orc)


# ---------------------------------------------------------------------------- golden / P1
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_golden_fixtures_gpu(ams, dtype):
    for name in ("spec_select_context_order.json", "spec_lookup_threshold.json"):
        fx = json.load(open(os.path.join(GOLDEN, name)))
        e = pad_d(np.array(fx["pool_emb"], np.float32))
        q = pad_d(np.array(fx["queries_emb"], np.float32))
        if dtype == "bf16":
            e, q = ams_gen.f32_to_bf16_bits(e), ams_gen.f32_to_bf16_bits(q)
        pj = np.array(fx["pool_joints"], np.float32)
        qj = np.array(fx["queries_joints"], np.float32)
        idx, s, hit = run_gpu(ams, e, pj, q, qj, fx["k"], fx["theta"], fx["gamma"], dtype)
        assert idx.tolist() == fx["expect"]["idx"], name
        assert hit.tolist() == fx["expect"]["hit"], name
    fx = json.load(open(os.path.join(GOLDEN, "gate_boundary.json")))
    e = pad_d(np.array(fx["pool_emb"], np.float32))
    q = pad_d(np.array(fx["queries_emb"], np.float32))
    if dtype == "bf16":
        e, q = ams_gen.f32_to_bf16_bits(e), ams_gen.f32_to_bf16_bits(q)
    for case in fx["cases"]:
        g = float(case["gamma"])
        idx, s, hit = run_gpu(ams, e, np.array(fx["pool_joints"], np.float32), q,
                              np.array(fx["queries_joints"], np.float32), fx["k"], fx["theta"], g, dtype)
        assert idx.tolist() == case["expect"]["idx"], g
        assert hit.tolist() == case["expect"]["hit"], g


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_p1_exhaustive_gpu(ams, dtype):
    rows = np.array(list(itertools.product([-1.0, 1.0], repeat=4)), np.float32)
    rng = np.random.Generator(np.random.PCG64(11))
    joints = rng.integers(-2, 3, (16, 2)).astype(np.float32)
    qj = np.array([[0, 0], [1, -1], [2, 2], [-2, 1]] * 4, np.float32)
    e = pad_d(rows)
    if dtype == "bf16":
        e = ams_gen.f32_to_bf16_bits(e)
    pool = ams.Pool(64, 2, 16, 16, 32, dtype=dtype)
    pool.append(to_dev(e), to_dev(joints), 16)
    for gamma in (0.0, 1.0, 2.0, INF):
        for k in (1, 3, 5, 16, 17):
            for theta in (1.0, 0.5, 0.0, -1.0):
                orc = oracle.match(e, joints, e, qj, k, theta, gamma)
                g = run_gpu(ams, e, joints, e, qj, k, theta, gamma, dtype, pool=pool)
                check_exact(*g, orc)   # every score is exact in both paths
    pool.close()


# ---------------------------------------------------------------------------- bf16 parity
SMALL = [
    # (config, M, Q) -- tile-spanning sizes with ragged tails, oracle finishes in seconds
    ("c2", 20011, 300),
    ("c3", 9001, 130),
    ("c4", 12345, 129),
    ("c5", 3001, 70),
]


@pytest.mark.parametrize("name,M,Q", SMALL)
@pytest.mark.parametrize("gated", [True, False])
def test_bf16_parity_small(ams, name, M, Q, gated):
    cfg = ams_gen.small_variant(name, M, Q)
    w = ams_gen.generate_host(cfg)
    gamma = cfg.gamma if gated else INF
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma)
    g = run_gpu(ams, w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma, "bf16")
    stats = check_bf16(*g, orc, cfg.theta, labels=w.labels)
    if gated:
        nd = w.labels >= 0
        assert np.array_equal(g[2].astype(bool), nd)   # P10 by construction
    assert stats["label_top1"] == 1.0


def test_bf16_host_vs_device_inputs_identical(ams):
    cfg = ams_gen.small_variant("c2", 5000, 64)
    w = ams_gen.generate_host(cfg)
    a = run_gpu(ams, w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, INF, "bf16")
    b = run_gpu(ams, w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, INF, "bf16", host_inputs=True)
    for x, y in zip(a, b):
        assert x.tobytes() == y.tobytes()


@pytest.mark.parametrize("nq", [37, 300])
@pytest.mark.parametrize("gated", [False, True])
def test_ties_across_splits_lowest_index(ams, nq, gated):
    """Exact ties (duplicate rows) spread over the whole pool: every merge level must
    keep (score desc, index asc); the shared admission bound admits equal scores."""
    rng = np.random.Generator(np.random.PCG64(77))
    d, J, M, k = 128, 7, 20000, 16
    base = ams_gen.f32_to_bf16_bits(rng.standard_normal((50, d)).astype(np.float32))
    emb = base[rng.integers(0, 50, M)]
    joints = np.zeros((M, J), np.float32)           # all rows eligible under any gate
    q = base[rng.integers(0, 50, nq)]
    qj = np.zeros((nq, J), np.float32)
    gamma = 0.3 if gated else INF
    orc = oracle.match(emb, joints, q, qj, k, 0.5, gamma)
    g = run_gpu(ams, emb, joints, q, qj, k, 0.5, gamma, "bf16")
    # the top-k are all exact duplicates of the query (score ~1, identical bits on GPU)
    assert np.array_equal(g[0], orc.idx)
    assert np.array_equal(g[2], orc.hit)
    assert np.abs(g[1] - orc.score).max() <= 2e-3


def test_plan_uses_cta_pairs_and_splits(ams):
    cfg = ams_gen.small_variant("c3", 30000, 600)
    w = ams_gen.generate_host(cfg)
    with ams.Pool(cfg.d, cfg.J, cfg.M, 1024, 32) as pool:
        pool.append(to_dev(w.emb), to_dev(w.joints))
        pool.match(to_dev(w.q_emb), to_dev(w.q_joints), cfg.k, cfg.theta, INF)
        plan = ams.ams_pool_last_plan(pool.handle)
        assert plan["kernel_id"] == 2 and plan["grid"] % 2 == 0 and plan["splits"] >= 1
        pool.match(to_dev(w.q_emb[:64]), to_dev(w.q_joints[:64]), cfg.k, cfg.theta, INF)
        plan = ams.ams_pool_last_plan(pool.handle)
        assert plan["kernel_id"] == 4 and plan["splits"] > 1 and plan["partials"] == 4 * plan["splits"]
        pool.match(to_dev(w.q_emb[:64]), to_dev(w.q_joints[:64]), cfg.k, cfg.theta, cfg.gamma)
        plan = ams.ams_pool_last_plan(pool.handle)
        # gated, one CTA per tile, KT <= 16: the 4 epilogue warps' lists are merged in the CTA
        assert plan["kernel_id"] == 4 and plan["splits"] > 1 and plan["partials"] == plan["splits"]
        ams.ams_pool_set_kernel_policy(pool.handle, 1)
        pool.match(to_dev(w.q_emb[:64]), to_dev(w.q_joints[:64]), cfg.k, cfg.theta, INF)
        plan = ams.ams_pool_last_plan(pool.handle)
        assert plan["kernel_id"] == 1 and plan["splits"] > 1
        torch.cuda.synchronize()


@pytest.mark.parametrize("k", [1, 9, 17, 33, 64])
@pytest.mark.parametrize("nq", [5, 200])
def test_every_topk_width_launches_and_matches(ams, k, nq):
    """KT in {8, 16, 32, 64} x single-CTA / CTA-pair kernels, plus the k > M padding."""
    cfg = ams_gen.small_variant("c2", 3000, nq)
    w = ams_gen.generate_host(cfg)
    for gamma in (INF, 1.5):
        orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, k, cfg.theta, gamma)
        g = run_gpu(ams, w.emb, w.joints, w.q_emb, w.q_joints, k, cfg.theta, gamma, "bf16", max_k=64)
        check_bf16(*g, orc, cfg.theta)
    e, j = w.emb[:40], w.joints[:40]
    orc = oracle.match(e, j, w.q_emb, w.q_joints, k, cfg.theta, INF)
    g = run_gpu(ams, e, j, w.q_emb, w.q_joints, k, cfg.theta, INF, "bf16", max_k=64)
    check_bf16(*g, orc, cfg.theta)


@pytest.mark.parametrize("nq", [64, 512])
def test_self_match_score_and_norms(ams, nq):
    """Pin P5 on the GPU: a query equal to a stored row with the same joints finds that
    row (or a lower-index duplicate) first with |s - 1| <= 1e-5 -- tight enough to catch
    an inverse norm that is off by more than a few ulps (fp32 sums over d = 1024 would
    not be) or a query/pool scale mix-up; the north_star tolerance is 2e-3."""
    cfg = ams_gen.small_variant("c3", 5000, nq)
    w = ams_gen.generate_host(cfg)
    rng = np.random.default_rng(nq)
    src = rng.choice(cfg.M, nq, replace=False)
    q, qj = w.emb[src], w.joints[src]
    for gamma in (0.3, INF):
        idx, score, hit = run_gpu(ams, w.emb, w.joints, q, qj, 4, 0.99, gamma, "bf16")
        assert np.all(idx[:, 0] <= src)
        assert np.all(np.abs(score[:, 0].astype(np.float64) - 1.0) <= 1e-5), np.abs(score[:, 0] - 1).max()
        assert np.all(hit == 1)


@pytest.mark.parametrize("M,nq,d", [(1, 1, 64), (31, 15, 64), (33, 17, 128), (1024, 64, 512), (1025, 100, 768),
                                    (5000, 33, 1024)])
@pytest.mark.parametrize("k", [1, 5, 16, 40])
def test_fp32_ungated_tile_kernel_bit_exact(ams, M, nq, d, k):
    """Ungated fp32 calls take the tiled exact kernel (plan id 6: 32-row x 16-query tiles,
    the canonical fmaf chain per pair); gated ones keep the thread-per-row kernel (plan id
    0).  Both byte-identical to the oracle, with duplicate rows (ties to the lower index)
    and ragged tiles."""
    rng = np.random.Generator(np.random.PCG64(M * 7 + nq + d + k))
    e = rng.standard_normal((M, d)).astype(np.float32)
    if M > 4:
        e[3] = e[1]
    qv = rng.standard_normal((nq, d)).astype(np.float32)
    j = rng.uniform(-1, 1, (M, 7)).astype(np.float32)
    qj = rng.uniform(-1, 1, (nq, 7)).astype(np.float32)
    with ams.Pool(d, 7, M, nq, 64, dtype="fp32") as pool:
        pool.append(to_dev(e), to_dev(j))
        for gamma, kid in ((INF, 6), (0.8, 0)):
            out = [t.cpu().numpy() for t in pool.match(to_dev(qv), to_dev(qj), k, 0.1, gamma)]
            torch.cuda.synchronize()
            assert ams.ams_pool_last_plan(pool.handle)["kernel_id"] == kid
            check_exact(*out, oracle.match(e, j, qv, qj, k, 0.1, gamma))


@pytest.mark.parametrize("M,nq,k", [(20011, 9, 5), (20011, 3, 32), (9000, 40, 16), (5000, 1, 1), (2100, 200, 32)])
def test_block_merge_rank_and_fallback_paths(ams, M, nq, k):
    """The block-per-query merge (nq < 8 x SMs, >= 64 partial lists, k <= 32) selects by
    rank over the list heads >= the kernels' bound; more than 512 such heads (an ungated
    fp32 call: no bound, every list full) takes the per-thread-list fallback.  fp32
    ungated calls with 626 / 282 / 157 / 66 lists cover both sides of the cap, byte-
    identical to the oracle, with duplicate rows (ties to the lower index)."""
    rng = np.random.Generator(np.random.PCG64(M + 31 * nq + k))
    d = 128
    e = rng.standard_normal((M, d)).astype(np.float32)
    e[5] = e[2]
    e[M - 1] = e[7]
    qv = rng.standard_normal((nq, d)).astype(np.float32)
    qv[0] = e[2]
    j = rng.uniform(-1, 1, (M, 7)).astype(np.float32)
    qj = rng.uniform(-1, 1, (nq, 7)).astype(np.float32)
    with ams.Pool(d, 7, M, nq, k, dtype="fp32") as pool:
        pool.append(to_dev(e), to_dev(j))
        out = [t.cpu().numpy() for t in pool.match(to_dev(qv), to_dev(qj), k, 0.2, INF)]
        torch.cuda.synchronize()
        plan = ams.ams_pool_last_plan(pool.handle)
        assert plan["kernel_id"] == 6 and plan["partials"] == (M + 31) // 32
        check_exact(*out, oracle.match(e, j, qv, qj, k, 0.2, INF))
