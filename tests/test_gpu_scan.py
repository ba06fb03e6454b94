"""GPU parity of the small-batch tcgen05 kernel (plan id 4: pool rows on the MMA M side,
the queries on N; nq <= 128 on one CTA per 256-row tile, 128 < nq <= 256 with k <= 8 on
a CTA pair) against the CPU oracle, and against the 128-query-tile
kernel (plan id 1) on the same inputs.

Covers every query-box size (NQ = 32, 64, 128 = round_up(nq, 32)),
KT in {8, 16, 32}, the JP = 4 / 8 / 16 joint strides, ragged pools (tiles of 256 rows
with a partial last tile, pools smaller than one tile), both gate modes, the
eligibility limits (k > 32 or round_up(nq, 32) * KT > 2048 fall back to plan id 1), exact ties across
splits, and appends between calls.  Expected values come only from oracle/.
"""
import numpy as np
import pytest

import ams_gen
import oracle
from tests.parity import check_bf16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
INF = float("inf")


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


def dev_t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.device("cuda", 0))


def scan_eligible(nq, k, gated=True, policy=0):
    """The library's rule: KT <= 32 and round_up(nq, 32) * KT <= 2048 (the per-lane
    register lists); nq <= 128 on one CTA per tile, 128 < nq <= 256 on a CTA pair with
    KT = 8 only, gated (ungated ones take the 256-query-tile kernel unless policy bit 3)."""
    KT = 8 if k <= 8 else 16 if k <= 16 else 32 if k <= 32 else 64
    if nq > 128:
        return nq <= 256 and KT == 8 and (gated or (policy & 8) != 0)
    return KT <= 32 and -(-nq // 32) * 32 * KT <= 2048


def run(ams, pool, q, qj, k, theta, gamma, policy=0):
    ams.ams_pool_set_kernel_policy(pool.handle, policy)
    out = pool.match(dev_t(q), dev_t(qj.astype(np.float32)), k, theta, gamma)
    torch.cuda.synchronize()
    plan = ams.ams_pool_last_plan(pool.handle)
    return tuple(t.cpu().numpy() for t in out), plan


@pytest.mark.parametrize("name,M", [("c2", 3001), ("c3", 2600), ("c5", 700)])
@pytest.mark.parametrize("nq", [1, 5, 16, 17, 33, 64, 100, 128, 129, 200, 256])
def test_scan_kernel_parity(ams, name, M, nq):
    cfg = ams_gen.small_variant(name, M, nq)
    w = ams_gen.generate_host(cfg)
    with ams.Pool(cfg.d, cfg.J, cfg.M, 256, 32) as pool:
        pool.append(dev_t(w.emb), dev_t(w.joints))
        for gamma in (cfg.gamma, 1.5, INF):
            orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma)
            g, plan = run(ams, pool, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma)
            assert plan["kernel_id"] == (4 if scan_eligible(nq, cfg.k, gamma != INF) else 1 if nq <= 128 else 2)
            stats = check_bf16(*g, orc, cfg.theta)
            if gamma == cfg.gamma:
                assert np.array_equal(g[2].astype(bool), w.labels >= 0)   # P10 by construction
            assert stats["queries"] == nq


@pytest.mark.parametrize("k", [1, 8, 9, 16, 17, 32])
@pytest.mark.parametrize("nq", [3, 64, 128])
def test_scan_kernel_topk_widths_and_fallback(ams, k, nq):
    """KT = 8/16/32 on both sides of the eligibility rule (plan id 4 vs 1)."""
    cfg = ams_gen.small_variant("c2", 4000, nq)
    w = ams_gen.generate_host(cfg)
    expect = {4} if scan_eligible(nq, k) else {1}
    with ams.Pool(cfg.d, cfg.J, cfg.M, 256, 64) as pool:
        pool.append(dev_t(w.emb), dev_t(w.joints))
        for gamma in (INF, 2.0):
            orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, k, cfg.theta, gamma)
            g, plan = run(ams, pool, w.q_emb, w.q_joints, k, cfg.theta, gamma)
            assert plan["kernel_id"] in expect
            check_bf16(*g, orc, cfg.theta)
        # k > 32 (KT = 64) always uses the 128-query-tile kernel
        orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, 40, cfg.theta, INF)
        g, plan = run(ams, pool, w.q_emb, w.q_joints, 40, cfg.theta, INF)
        assert plan["kernel_id"] == 1
        check_bf16(*g, orc, cfg.theta)


@pytest.mark.parametrize("M", [1, 37, 255, 256, 257, 513])
@pytest.mark.parametrize("nq", [20, 150])
def test_scan_kernel_tiny_and_ragged_pools(ams, M, nq):
    cfg = ams_gen.small_variant("c3", M, nq)
    w = ams_gen.generate_host(cfg)
    with ams.Pool(cfg.d, cfg.J, cfg.M, 256, 16) as pool:
        pool.append(dev_t(w.emb), dev_t(w.joints))
        for k in ((1, 16) if nq <= 128 else (1, 8)):
            for gamma in (0.3, INF):
                orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, k, cfg.theta, gamma)
                g, plan = run(ams, pool, w.q_emb, w.q_joints, k, cfg.theta, gamma, policy=8)
                assert plan["kernel_id"] == 4
                check_bf16(*g, orc, cfg.theta)


def test_scan_kernel_matches_tile_kernel(ams):
    """Both kernels on the same pool and queries: same valid counts, index sets where
    the oracle's gaps are wide, scores within the bf16 tolerance of each other."""
    cfg = ams_gen.small_variant("c3", 9001, 64)
    w = ams_gen.generate_host(cfg)
    with ams.Pool(cfg.d, cfg.J, cfg.M, 256, 16) as pool:
        pool.append(dev_t(w.emb), dev_t(w.joints))
        for gamma in (cfg.gamma, INF):
            orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma)
            a, pa = run(ams, pool, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma, policy=0)
            b, pb = run(ams, pool, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma, policy=1)
            assert pa["kernel_id"] == 4 and pb["kernel_id"] == 1
            check_bf16(*a, orc, cfg.theta)
            check_bf16(*b, orc, cfg.theta)
            assert np.array_equal(a[0] >= 0, b[0] >= 0)
            v = a[0] >= 0
            assert np.abs(a[1][v] - b[1][v]).max(initial=0.0) <= 2e-3


@pytest.mark.parametrize("gated", [False, True])
def test_scan_kernel_exact_ties_lowest_index(ams, gated):
    """50 distinct rows repeated over 20,000 (many splits): every query's top-k are exact
    duplicates of it; the lists must keep (score desc, index asc) through the per-warp
    lists, the shared bound (ties admitted) and the merge."""
    rng = np.random.Generator(np.random.PCG64(78))
    d, J, M, k, nq = 128, 7, 20000, 16, 64
    base = ams_gen.f32_to_bf16_bits(rng.standard_normal((50, d)).astype(np.float32))
    emb = base[rng.integers(0, 50, M)]
    joints = np.zeros((M, J), np.float32)
    q = base[rng.integers(0, 50, nq)]
    qj = np.zeros((nq, J), np.float32)
    gamma = 0.3 if gated else INF
    orc = oracle.match(emb, joints, q, qj, k, 0.5, gamma)
    with ams.Pool(d, J, M, nq, k) as pool:
        pool.append(dev_t(emb), dev_t(joints))
        g, plan = run(ams, pool, q, qj, k, 0.5, gamma)
    assert plan["kernel_id"] == 4 and plan["splits"] > 10
    assert np.array_equal(g[0], orc.idx)
    assert np.array_equal(g[2], orc.hit)
    assert np.abs(g[1] - orc.score).max() <= 2e-3


def test_scan_kernel_gate_boundary_and_appends(ams):
    """Integer joints make ds exact: rows at ds == gamma^2 are eligible, ds == gamma^2 + 1
    are not; appends between calls are visible to the next call."""
    rng = np.random.Generator(np.random.PCG64(79))
    d, J, k = 64, 3, 8
    M0, M1 = 700, 300
    emb = ams_gen.f32_to_bf16_bits(rng.standard_normal((M0 + M1, d)).astype(np.float32))
    joints = rng.integers(-3, 4, (M0 + M1, J)).astype(np.float32)
    nq = 24
    q = ams_gen.f32_to_bf16_bits(rng.standard_normal((nq, d)).astype(np.float32))
    qj = rng.integers(-3, 4, (nq, J)).astype(np.float32)
    with ams.Pool(d, J, M0 + M1, nq, k) as pool:
        pool.append(dev_t(emb[:M0]), dev_t(joints[:M0]))
        for gamma in (0.0, 1.0, 2.0):
            orc = oracle.match(emb[:M0], joints[:M0], q, qj, k, 0.0, gamma)
            g, plan = run(ams, pool, q, qj, k, 0.0, gamma)
            assert plan["kernel_id"] == 4
            check_bf16(*g, orc, 0.0)
        pool.append(dev_t(emb[M0:]), dev_t(joints[M0:]))
        for gamma in (1.0, INF):
            orc = oracle.match(emb, joints, q, qj, k, 0.0, gamma)
            g, plan = run(ams, pool, q, qj, k, 0.0, gamma)
            check_bf16(*g, orc, 0.0)


@pytest.mark.parametrize("nq", [1, 7, 63, 64, 65, 255, 256])
def test_survey_batch_and_k_grid(ams, nq):
    """SURVEY.md 4, tier 2: k in {1, 5, 16, 32} x nq in {1, 7, 63, 64, 65, 255, 256} on a
    pool that is not a multiple of the tile, gated and ungated, against the oracle --
    whichever kernel the plan picks (small-batch on one CTA or a CTA pair, or the
    128/256-query-tile kernel)."""
    cfg = ams_gen.small_variant("c2", 3001, nq)
    w = ams_gen.generate_host(cfg)
    with ams.Pool(cfg.d, cfg.J, cfg.M, 256, 32) as pool:
        pool.append(dev_t(w.emb), dev_t(w.joints))
        for k in (1, 5, 16, 32):
            for gamma in (cfg.gamma, INF):
                orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, k, cfg.theta, gamma)
                g, plan = run(ams, pool, w.q_emb, w.q_joints, k, cfg.theta, gamma)
                assert plan["kernel_id"] == (4 if scan_eligible(nq, k, gamma != INF) else 1 if nq <= 128 else 2)
                check_bf16(*g, orc, cfg.theta)


@pytest.mark.parametrize("M", [1, 255, 256, 257, 511, 513, 767, 769, 5000, 20011])
@pytest.mark.parametrize("nq", [129, 200, 256])
def test_wide_pair_matches_narrow_pair_and_oracle(ams, M, nq):
    """CTA pairs, 129-256 queries: the wide mode (policy bit 2: two 256-row tiles per
    pipeline stage, single-buffered accumulators) against the oracle and byte-for-byte
    against the narrow default -- same MMA shape and K order per element, so the same bits.  Pools
    with an odd tile count leave the last super-tile half past the pool (no loads, no
    scores); tiny pools give empty splits."""
    cfg = ams_gen.small_variant("c3", M, nq)
    w = ams_gen.generate_host(cfg)
    with ams.Pool(cfg.d, cfg.J, cfg.M, 256, 8) as pool:
        pool.append(dev_t(w.emb), dev_t(w.joints))
        for k in (1, 8):
            for gamma in (0.3, 2.5, INF):
                orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, k, cfg.theta, gamma)
                a, pa = run(ams, pool, w.q_emb, w.q_joints, k, cfg.theta, gamma, policy=4 | 8)
                b, pb = run(ams, pool, w.q_emb, w.q_joints, k, cfg.theta, gamma, policy=8)
                assert pa["kernel_id"] == 4 and pb["kernel_id"] == 4
                check_bf16(*a, orc, cfg.theta)
                for x, y in zip(a, b):
                    assert x.tobytes() == y.tobytes()


def test_wide_pair_appends_between_calls(ams):
    """Appends move L past super-tile boundaries between calls (the split plan and the
    half-empty last super-tile change every call)."""
    cfg = ams_gen.small_variant("c5", 3000, 180)
    w = ams_gen.generate_host(cfg)
    with ams.Pool(cfg.d, cfg.J, cfg.M, 256, 8) as pool:
        done = 0
        for step in (300, 212, 256, 1000, 1232):
            pool.append(dev_t(w.emb[done:done + step]), dev_t(w.joints[done:done + step]))
            done += step
            orc = oracle.match(w.emb[:done], w.joints[:done], w.q_emb, w.q_joints, 8, cfg.theta, INF)
            for pol in (8, 4 | 8):
                a, pa = run(ams, pool, w.q_emb, w.q_joints, 8, cfg.theta, INF, policy=pol)
                assert pa["kernel_id"] == 4
                check_bf16(*a, orc, cfg.theta)


def test_ungated_pair_batches_route_to_tile_kernel(ams):
    """Ungated 129-256-query batches take the 256-query-tile kernel by default (plan id 2),
    the small-batch CTA pairs with policy bit 3; both agree with the oracle."""
    cfg = ams_gen.small_variant("c3", 4001, 200)
    w = ams_gen.generate_host(cfg)
    with ams.Pool(cfg.d, cfg.J, cfg.M, 256, 8) as pool:
        pool.append(dev_t(w.emb), dev_t(w.joints))
        orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, 8, cfg.theta, INF)
        for pol, kid in ((0, 2), (8, 4)):
            g, plan = run(ams, pool, w.q_emb, w.q_joints, 8, cfg.theta, INF, policy=pol)
            assert plan["kernel_id"] == kid
            check_bf16(*g, orc, cfg.theta)
        g, plan = run(ams, pool, w.q_emb, w.q_joints, 8, cfg.theta, 0.3)   # gated: the pairs
        assert plan["kernel_id"] == 4
