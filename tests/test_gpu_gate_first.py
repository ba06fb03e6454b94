"""Gate-first sparse variant (ams_match_gate_first) vs the oracle."""
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


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(ams, w, k, theta, gamma, gate_first, max_k=None):
    M, d = w.emb.shape
    with ams.Pool(d, w.joints.shape[1], max(M, 1), w.q_emb.shape[0], max_k or k) as pool:
        pool.append(T(w.emb), T(w.joints))
        out = pool.match(T(w.q_emb), T(w.q_joints), k, theta, gamma, gate_first=gate_first)
        torch.cuda.synchronize()
        if gate_first:
            assert ams.ams_pool_last_plan(pool.handle)["kernel_id"] == 3
        return [t.cpu().numpy() for t in out]


@pytest.mark.parametrize("name,M,Q", [("c2", 20011, 300), ("c3", 9001, 130), ("c4", 12345, 129),
                                      ("c5", 3001, 70)])
@pytest.mark.parametrize("gamma", [0.3, 1.2])
def test_gate_first_parity_small(ams, name, M, Q, gamma):
    cfg = ams_gen.small_variant(name, M, Q)
    w = ams_gen.generate_host(cfg)
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma, mode="B")
    g = run(ams, w, cfg.k, cfg.theta, gamma, True)
    check_bf16(*g, orc, cfg.theta)
    # same eligible sets and ranking as the dense path
    dense = run(ams, w, cfg.k, cfg.theta, gamma, False)
    assert np.array_equal(g[0] >= 0, dense[0] >= 0)


@pytest.mark.parametrize("gamma", [20.0, INF])
def test_gate_first_bucket_overflow_is_exact(ams, gamma):
    """Every row eligible: every bucket overflows and the exact per-query scan runs."""
    cfg = ams_gen.small_variant("c2", 1500, 40)
    w = ams_gen.generate_host(cfg)
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma)
    g = run(ams, w, cfg.k, cfg.theta, gamma, True)
    check_bf16(*g, orc, cfg.theta)


@pytest.mark.parametrize("nq", [1, 2, 16, 17, 32, 33, 64, 65, 128, 129, 256])
@pytest.mark.parametrize("gamma", [0.6, INF])
def test_gate_first_batch_shapes(ams, nq, gamma):
    """Batch-size dispatch of the gate scan: <= 16 queries take the row-parallel kernel
    (thread per row, exact gate against every query), larger batches the warp kernel with
    32 / 64 / 128 / 256 queries per block (warps split the rows when fewer than 256).  A
    ragged pool (rows past the last full tile) and gamma = inf (every row eligible: with
    k = 5 the buckets overflow and the exact scan runs) for each side of every boundary."""
    cfg = ams_gen.small_variant("c5", 3001, nq)
    w = ams_gen.generate_host(cfg)
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma)
    g = run(ams, w, cfg.k, cfg.theta, gamma, True)
    check_bf16(*g, orc, cfg.theta)


@pytest.mark.parametrize("nq,gamma", [(17, 0.3), (40, 0.8), (300, 0.3), (1024, 0.2), (1025, 0.3)])
def test_gate_first_binned_snapshot_and_tail(ams, nq, gamma):
    """Gated batches of 17..1024 queries are staged in joint-0 bins; on a pool of >= 64 K
    rows the first call builds the joint-0 row snapshot and scans it with warp-uniform
    windows, and rows appended afterwards (below the rebuild threshold) are scanned by the
    pair-dealing kernel.  1025 queries: the 2-D query order and the block kernel over the
    snapshot and the appended tail.  Both calls against the oracle, the second after a
    5,000-row append."""
    cfg = ams_gen.small_variant("c2", 75000, nq)
    w = ams_gen.generate_host(cfg)
    M0 = 70000
    with ams.Pool(cfg.d, cfg.J, cfg.M, nq, cfg.k) as pool:
        pool.append(T(w.emb[:M0]), T(w.joints[:M0]))
        out = [t.cpu().numpy() for t in pool.match(T(w.q_emb), T(w.q_joints), cfg.k, cfg.theta, gamma,
                                                    gate_first=True)]
        torch.cuda.synchronize()
        check_bf16(*out, oracle.match(w.emb[:M0], w.joints[:M0], w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma),
                   cfg.theta)
        pool.append(T(w.emb[M0:]), T(w.joints[M0:]))
        out = [t.cpu().numpy() for t in pool.match(T(w.q_emb), T(w.q_joints), cfg.k, cfg.theta, gamma,
                                                    gate_first=True)]
        torch.cuda.synchronize()
        assert ams.ams_pool_last_plan(pool.handle)["kernel_id"] == 3
    check_bf16(*out, oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma), cfg.theta)


@pytest.mark.parametrize("M,nq", [(3001, 100), (20011, 1024)])
def test_gate_first_binned_small_pool(ams, M, nq):
    """Pools below the snapshot threshold: the binned batch goes to the pair-dealing kernel
    over the whole pool."""
    cfg = ams_gen.small_variant("c2", M, nq)
    w = ams_gen.generate_host(cfg)
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, 0.5)
    check_bf16(*run(ams, w, cfg.k, cfg.theta, 0.5, True), orc, cfg.theta)


def test_gate_first_ties_and_padding(ams):
    rng = np.random.Generator(np.random.PCG64(5))
    d, J, M = 128, 7, 3000
    base = ams_gen.f32_to_bf16_bits(rng.standard_normal((20, d)).astype(np.float32))
    emb = base[rng.integers(0, 20, M)]
    joints = np.where(rng.random((M, J)) < 0.5, 0.0, 3.0).astype(np.float32)   # half the rows near 0
    q = base[rng.integers(0, 20, 50)]
    qj = np.zeros((50, J), np.float32)
    w = ams_gen.Workload(ams_gen.CONFIGS["c2"], emb, joints, q, qj, -np.ones(50, np.int64))
    for k in (5, 40):
        orc = oracle.match(emb, joints, q, qj, k, 0.5, 0.3)
        g = run(ams, w, k, 0.5, 0.3, True, max_k=64)
        assert np.array_equal(g[0], orc.idx)        # exact ties -> lowest indices
        assert np.array_equal(g[2], orc.hit)


def test_gate_first_c3_full_size_sampled(ams):
    cfg = ams_gen.CONFIGS["c3"]
    dev = torch.device("cuda", 0)
    pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k)
    q, qj, labels, host_e, host_j = ams_gen.build_device_workload(
        cfg, dev, lambda e, j, n: pool.append(e, j, n), host_copy=True)
    gi, gs, gh = (t.cpu().numpy() for t in pool.match(q, qj, cfg.k, cfg.theta, cfg.gamma, gate_first=True))
    pool.close()
    lab = labels.cpu().numpy()
    nd = lab >= 0
    assert np.array_equal(gh.astype(bool), nd) and np.array_equal(gi[nd, 0], lab[nd])
    sel = np.arange(0, cfg.Q, cfg.Q // 1024)
    qn = q.view(torch.int16).cpu().numpy().view(np.uint16)
    orc = oracle.match(host_e, host_j, qn[sel], qj.cpu().numpy()[sel], cfg.k, cfg.theta, cfg.gamma, mode="B")
    check_bf16(gi[sel], gs[sel], gh[sel], orc, cfg.theta)
