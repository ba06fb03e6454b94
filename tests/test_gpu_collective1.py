"""The world > 1 code path of ams_match on ONE GPU: a pool created with world == 1 and
an NCCL unique id builds a 1-rank communicator and runs the shard merge, the
ncclAllGather of the [nq, k] shard lists, and the final G-way merge kernel (and, once
enabled, the fused peer-exchange kernels with G = 1) -- the same host and device code
as a multi-GPU run, minus the cross-GPU transfers.  Results must equal the oracle
(north_star tolerances) and be bit-identical to a plain world == 1 pool.

No rank ever waits on another GPU's kernel here (G = 1), so this stays within the
one-GPU testing rule of the profiling guide.
"""
import math

import numpy as np
import pytest

import ams_gen
import oracle
from tests.parity import check_bf16, check_exact

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(ams, w, cfg, k, gamma, collective, peer=False, gate_first=False, block=0):
    nid = ams.ams_get_nccl_unique_id() if collective else None
    dt = "bf16" if cfg.dtype == "bf16" else "fp32"
    pool = ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, k, dtype=dt, nccl_id=nid, shard_block=block)
    try:
        if peer:
            ams.ams_pool_enable_peer_exchange(pool.handle)
        pool.append(T(w.emb), T(w.joints))
        res = []
        for _ in range(2):   # two calls: the peer path alternates its parity slots
            out = pool.match(T(w.q_emb), T(w.q_joints), k, cfg.theta, gamma, gate_first=gate_first)
            torch.cuda.synchronize()
            res.append([t.cpu().numpy() for t in out])
        for a, b in zip(res[0], res[1]):
            np.testing.assert_array_equal(a, b)
        return res[1]
    finally:
        pool.close()


@pytest.mark.parametrize("gamma", [0.3, math.inf])
@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("name,nq", [("c2", 600), ("c2", 64), ("c5", 200)])   # CTA-pair tiles; small-batch kernel
def test_collective_path_bf16(ams, gamma, peer, name, nq):
    cfg = ams_gen.small_variant(name, 7000, nq)
    w = ams_gen.generate_host(cfg)
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma)
    got = run(ams, w, cfg, cfg.k, gamma, collective=True, peer=peer)
    check_bf16(*got, orc, cfg.theta)
    ref = run(ams, w, cfg, cfg.k, gamma, collective=False)
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("peer", [False, True])
def test_collective_path_gate_first(ams, peer):
    cfg = ams_gen.small_variant("c2", 5000, 300)
    w = ams_gen.generate_host(cfg)
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, cfg.gamma)
    got = run(ams, w, cfg, cfg.k, cfg.gamma, collective=True, peer=peer, gate_first=True)
    check_bf16(*got, orc, cfg.theta)


@pytest.mark.parametrize("gamma", [0.3, math.inf])
def test_collective_path_fp32_bit_exact(ams, gamma):
    cfg = ams_gen.CONFIGS["c1"]
    w = ams_gen.generate_host(cfg)
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma)
    check_exact(*run(ams, w, cfg, cfg.k, gamma, collective=True), orc)
    check_exact(*run(ams, w, cfg, cfg.k, gamma, collective=True, peer=True), orc)


def test_peer_exchange_needs_a_communicator(ams):
    with ams.Pool(64, 2, 100, 8, 4) as pool:
        with pytest.raises(ams.AmsError) as e:
            ams.ams_pool_enable_peer_exchange(pool.handle)
        assert e.value.status == 6   # AMS_ERR_UNSUPPORTED
