"""GPU parity of the joint-0-ordered gated path (ams_capi.cu kSortMinQueries,
ams_match_tc.cu epi_chunk_sorted) against the oracle.

Gated bf16 batches of >= 129 queries are staged in joint-0 order and the epilogue
rejects pool columns for a whole warp at once from the warp's joint-0 interval.  The
configs' gate passes almost nothing (reading R14), so these cases use joints drawn
from narrow ranges and integer joints with integer gate radii, so that many pairs are
eligible, many sit exactly on the gate boundary (ds == g2), and the warp-level test
must keep every one of them.  Expected values come only from oracle/.
"""
import numpy as np
import pytest

import ams_gen
import oracle
from tests.parity import check_bf16
from tests.test_gpu_parity import run_gpu

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
INF = float("inf")


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


def emb_bits(rng, n, d):
    x = rng.standard_normal((n, d)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return ams_gen.f32_to_bf16_bits(x)


def near_dups(rng, src_bits, sigma):
    x = ams_gen.bf16_bits_to_f32(src_bits)
    x = x + sigma * rng.standard_normal(x.shape).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return ams_gen.f32_to_bf16_bits(x)


@pytest.mark.parametrize("J,M,nq,spread,gamma", [
    (1, 3001, 129, 1.0, 0.05),      # J = 1: the warp test is the whole gate
    (3, 5000, 300, 0.5, 0.3),
    (7, 4097, 777, 0.4, 0.3),
    (14, 2600, 2048, 0.15, 0.35),
    (7, 20000, 4100, 3.14159, 0.3),  # the configs' joint law, many tiles
])
def test_sorted_gated_dense_gate(ams, J, M, nq, spread, gamma):
    rng = np.random.default_rng(1000 + J + nq)
    d = 128
    pe = emb_bits(rng, M, d)
    pj = rng.uniform(-spread, spread, (M, J)).astype(np.float32)
    src = rng.integers(0, M, nq // 2)
    q = np.concatenate([near_dups(rng, pe[src], 0.05 / np.sqrt(d)), emb_bits(rng, nq - nq // 2, d)])
    qj = np.concatenate([pj[src] + rng.normal(0, 0.02, (src.size, J)).astype(np.float32),
                         rng.uniform(-spread, spread, (nq - nq // 2, J)).astype(np.float32)])
    k, theta = 10, 0.9
    orc = oracle.match(pe, pj, q, qj, k, theta, gamma)
    assert orc.nelig.mean() > 0.5 or spread > 3, "case must exercise the gate"
    g = run_gpu(ams, pe, pj, q, qj, k, theta, gamma, "bf16")
    check_bf16(*g, orc, theta)


@pytest.mark.parametrize("host_inputs", [False, True])
def test_sorted_gate_boundary_integer_joints(ams, host_inputs):
    """Integer joints and gamma = 1: ds is an exact integer and every pair with ds == 1
    is eligible (reading R3, inclusive).  Joint 0 takes few values, so many warps hold
    queries with equal r_0 and pool columns sit exactly at wlo - 1 / whi + 1."""
    rng = np.random.default_rng(7)
    M, d, J, nq = 2000, 64, 4, 640
    pe = emb_bits(rng, M, d)
    pj = rng.integers(-2, 3, (M, J)).astype(np.float32)
    q = emb_bits(rng, nq, d)
    qj = rng.integers(-2, 3, (nq, J)).astype(np.float32)
    for gamma in (0.0, 1.0, 2.0):
        orc = oracle.match(pe, pj, q, qj, 16, 0.5, gamma)
        g = run_gpu(ams, pe, pj, q, qj, 16, 0.5, gamma, "bf16", host_inputs=host_inputs)
        check_bf16(*g, orc, 0.5)


def test_sorted_degenerate_joint0(ams):
    """All queries share joint 0 (zero span: one bin), then a span of 1e30 (bins
    collapse at the ends): the order is only a heuristic, results must not change."""
    rng = np.random.default_rng(11)
    M, d, J, nq = 3000, 64, 2, 300
    pe = emb_bits(rng, M, d)
    pj = rng.uniform(-0.5, 0.5, (M, J)).astype(np.float32)
    q = emb_bits(rng, nq, d)
    qj = rng.uniform(-0.5, 0.5, (nq, J)).astype(np.float32)
    qj[:, 0] = 0.125
    orc = oracle.match(pe, pj, q, qj, 8, 0.5, 0.4)
    check_bf16(*run_gpu(ams, pe, pj, q, qj, 8, 0.5, 0.4, "bf16"), orc, 0.5)
    qj[0, 0], qj[1, 0] = 1e30, -1e30
    orc = oracle.match(pe, pj, q, qj, 8, 0.5, 0.4)
    check_bf16(*run_gpu(ams, pe, pj, q, qj, 8, 0.5, 0.4, "bf16"), orc, 0.5)


def test_sorted_matches_unsorted_batches(ams):
    """The same queries matched as one sorted batch (nq >= 129) and as unsorted batches
    of <= 128: both agree with the oracle, and with each other on every index."""
    rng = np.random.default_rng(5)
    M, d, J, nq = 6000, 256, 7, 512
    pe = emb_bits(rng, M, d)
    pj = rng.uniform(-0.4, 0.4, (M, J)).astype(np.float32)
    src = rng.integers(0, M, nq)
    q = near_dups(rng, pe[src], 0.3 / np.sqrt(d))
    qj = pj[src] + rng.normal(0, 0.05, (nq, J)).astype(np.float32)
    orc = oracle.match(pe, pj, q, qj, 12, 0.95, 0.3)
    with ams.Pool(d, J, M, nq, 12) as pool:
        pool.append(torch.from_numpy(pe).cuda(), torch.from_numpy(pj).cuda())
        whole = [t.cpu().numpy() for t in pool.match(torch.from_numpy(q).cuda(), torch.from_numpy(qj).cuda(),
                                                     12, 0.95, 0.3)]
        parts = [[t.cpu().numpy() for t in pool.match(torch.from_numpy(q[a:a + 100]).cuda(),
                                                      torch.from_numpy(qj[a:a + 100]).cuda(), 12, 0.95, 0.3)]
                 for a in range(0, nq, 100)]
    check_bf16(*whole, orc, 0.95)
    for i in range(3):
        np.testing.assert_array_equal(whole[i], np.concatenate([p[i] for p in parts]))


@pytest.mark.parametrize("J,M,nq,spread,gamma", [
    (1, 3001, 129, 1.0, 0.05),
    (7, 4097, 777, 0.4, 0.3),
    (14, 2600, 2048, 0.15, 0.35),
    (7, 20000, 4100, 3.14159, 0.3),
])
def test_sorted_gate_first(ams, J, M, nq, spread, gamma):
    """The gate-first variant takes the same joint-0 order (warp-level row test in
    gate_scan_kernel, outputs scattered back by score_kernel)."""
    rng = np.random.default_rng(2000 + J + nq)
    d = 128
    pe = emb_bits(rng, M, d)
    pj = rng.uniform(-spread, spread, (M, J)).astype(np.float32)
    src = rng.integers(0, M, nq // 2)
    q = np.concatenate([near_dups(rng, pe[src], 0.05 / np.sqrt(d)), emb_bits(rng, nq - nq // 2, d)])
    qj = np.concatenate([pj[src] + rng.normal(0, 0.02, (src.size, J)).astype(np.float32),
                         rng.uniform(-spread, spread, (nq - nq // 2, J)).astype(np.float32)])
    orc = oracle.match(pe, pj, q, qj, 10, 0.9, gamma)
    with ams.Pool(d, J, M, nq, 10) as pool:
        pool.append(torch.from_numpy(pe).cuda(), torch.from_numpy(pj).cuda())
        g = [t.cpu().numpy() for t in pool.match(torch.from_numpy(q).cuda(), torch.from_numpy(qj).cuda(), 10, 0.9,
                                                 gamma, gate_first=True)]
    check_bf16(*g, orc, 0.9)


def test_host_staging_pipeline(ams):
    """Back-to-back calls with host inputs and no synchronisation in between: the
    double-buffered staging (copy stream + events) must hand every call its own
    queries.  Mixed sizes exercise both the sorted (>= 129) and plain staging."""
    rng = np.random.default_rng(21)
    M, d, J = 3000, 128, 7
    pe = emb_bits(rng, M, d)
    pj = rng.uniform(-0.5, 0.5, (M, J)).astype(np.float32)
    sizes = [300, 64, 1000, 129, 5, 777]
    qs = [emb_bits(rng, n, d) for n in sizes]
    qjs = [rng.uniform(-0.5, 0.5, (n, J)).astype(np.float32) for n in sizes]
    with ams.Pool(d, J, M, max(sizes), 10) as pool:
        pool.append(torch.from_numpy(pe).cuda(), torch.from_numpy(pj).cuda())
        torch.cuda.synchronize()
        hq = [torch.from_numpy(q).pin_memory() for q in qs]
        hj = [torch.from_numpy(j).pin_memory() for j in qjs]
        outs = [pool.match(a, b, 10, 0.9, 0.3) for a, b in zip(hq, hj)]
        torch.cuda.synchronize()
    for q, qj, o in zip(qs, qjs, outs):
        orc = oracle.match(pe, pj, q, qj, 10, 0.9, 0.3)
        check_bf16(*[t.cpu().numpy() for t in o], orc, 0.9)


def test_gate_first_joint_index_and_tail(ams):
    """Pools of >= 64 K local rows: sorted gate-first batches scan the joint-0 index
    (bucket-sorted snapshot) for the rows within gamma of each block's joint-0 interval,
    plus the rows appended since the snapshot in plain order; the snapshot is rebuilt
    once that tail exceeds max(64 K, L/32).  Dense-gate joints (many eligible rows per
    query, many near bin and gate boundaries) against the oracle after each stage:
    fresh index, index + tail, rebuilt index."""
    rng = np.random.default_rng(77)
    d, J, k = 64, 3, 12
    sizes = [70000, 20000, 60000]
    M = sum(sizes)
    pe = emb_bits(rng, M, d)
    pj = rng.uniform(-0.6, 0.6, (M, J)).astype(np.float32)
    pj[::97, 0] = np.round(pj[::97, 0], 1)   # exact ties in joint 0 at bin-friendly values
    nq = 300
    q = emb_bits(rng, nq, d)
    qj = rng.uniform(-0.6, 0.6, (nq, J)).astype(np.float32)
    qj[::7, 0] = np.round(qj[::7, 0], 1)
    gamma = 0.12
    with ams.Pool(d, J, M, nq, k) as pool:
        lo = 0
        for n in sizes:
            pool.append(torch.from_numpy(pe[lo:lo + n]).cuda(), torch.from_numpy(pj[lo:lo + n]).cuda())
            lo += n
            g = [t.cpu().numpy() for t in pool.match(torch.from_numpy(q).cuda(), torch.from_numpy(qj).cuda(), k,
                                                     0.5, gamma, gate_first=True)]
            orc = oracle.match(pe[:lo], pj[:lo], q, qj, k, 0.5, gamma)
            assert orc.nelig.mean() > 20, "case must exercise the gate"
            check_bf16(*g, orc, 0.5)
