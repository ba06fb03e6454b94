"""Sharding on one GPU (pin P8 on the GPU path).

The multi-GPU protocol is: every rank computes the exact top-k of its shard, the
lists are all-gathered (NCCL), and the final k-way merge kernel produces the result on
every rank.  With one GPU we run the same protocol with G single-GPU pools ("virtual
shards", no kernels waiting on one another) and the same merge kernel
(ams_merge_topk), and require outputs BIT-IDENTICAL to the unsharded pool: a pair's
fp32 score depends only on its own K-reduction, never on its tile position.
"""
import numpy as np
import pytest

import ams_gen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
INF = float("inf")


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


def dev():
    return torch.device("cuda", 0)


@pytest.mark.parametrize("G,kin,k", [(1, 5, 5), (2, 16, 10), (3, 16, 16), (8, 32, 32), (5, 8, 3)])
def test_merge_topk_matches_oracle_merge(ams, G, kin, k):
    rng = np.random.Generator(np.random.PCG64(G * 100 + kin))
    nq = 257
    # scores from a small set so that ties across lists are common; ids unique per query
    s = np.sort(rng.choice(np.linspace(-1, 1, 9).astype(np.float32), (G, nq, kin)), axis=2)[:, :, ::-1]
    ids = np.empty((G, nq, kin), np.int64)
    for i in range(nq):
        perm = rng.permutation(G * kin * 4)[: G * kin].reshape(G, kin)
        ids[:, i, :] = perm
    # each list ordered by (score desc, id asc); pad some tails with (-inf, -1)
    for g in range(G):
        for i in range(nq):
            o = np.lexsort((ids[g, i], -s[g, i]))
            s[g, i], ids[g, i] = s[g, i][o], ids[g, i][o]
            cut = rng.integers(0, kin + 1)
            s[g, i, cut:] = -np.inf
            ids[g, i, cut:] = -1
    s = np.ascontiguousarray(s)
    orc = oracle.merge(s.astype(np.float64), ids, k, 0.25)
    out_i = torch.empty(nq, k, dtype=torch.int64, device=dev())
    out_s = torch.empty(nq, k, dtype=torch.float32, device=dev())
    out_h = torch.empty(nq, dtype=torch.uint8, device=dev())
    ams.ams_merge_topk(torch.from_numpy(s).to(dev()), torch.from_numpy(ids).to(dev()), G, nq, kin, k, 0.25,
                       out_i, out_s, out_h)
    torch.cuda.synchronize()
    assert np.array_equal(out_i.cpu().numpy(), orc.idx)
    assert out_s.cpu().numpy().tobytes() == orc.score.tobytes()
    assert np.array_equal(out_h.cpu().numpy(), orc.hit)


def _pool_run(ams, emb, joints, q, qj, k, theta, gamma, cap=None):
    with ams.Pool(emb.shape[1], joints.shape[1], cap or max(len(emb), 1), q.shape[0], k) as pool:
        if len(emb):
            pool.append(torch.from_numpy(emb).to(dev()), torch.from_numpy(joints).to(dev()))
        out = pool.match(torch.from_numpy(q).to(dev()), torch.from_numpy(qj).to(dev()), k, theta, gamma)
        torch.cuda.synchronize()
        return [t.clone() for t in out]


@pytest.mark.parametrize("G,block", [(2, 0), (4, 256), (8, 0), (3, 1000)])
@pytest.mark.parametrize("nq", [64, 300])
def test_virtual_shards_bit_identical(ams, G, block, nq):
    cfg = ams_gen.small_variant("c4", 24007, nq)
    w = ams_gen.generate_host(cfg)
    for gamma in (INF, cfg.gamma):
        full = _pool_run(ams, w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma)
        owner = np.array([ams.ams_shard_locate(cfg.M, G, block, o)[0] for o in range(cfg.M)])
        lists_s, lists_i = [], []
        for g in range(G):
            rows = np.nonzero(owner == g)[0]
            li, ls, _ = _pool_run(ams, w.emb[rows], w.joints[rows], w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma,
                                  cap=max(len(rows), 1))
            li = li.cpu().numpy()
            gi = np.where(li >= 0, rows[np.clip(li, 0, None)], -1)   # local -> global ordinal
            lists_i.append(gi)
            lists_s.append(ls.cpu().numpy())
        S = torch.from_numpy(np.ascontiguousarray(np.stack(lists_s))).to(dev())
        I = torch.from_numpy(np.ascontiguousarray(np.stack(lists_i))).to(dev())
        oi = torch.empty(nq, cfg.k, dtype=torch.int64, device=dev())
        os_ = torch.empty(nq, cfg.k, dtype=torch.float32, device=dev())
        oh = torch.empty(nq, dtype=torch.uint8, device=dev())
        ams.ams_merge_topk(S, I, G, nq, cfg.k, cfg.k, cfg.theta, oi, os_, oh)
        torch.cuda.synchronize()
        assert torch.equal(oi, full[0]), gamma
        assert os_.cpu().numpy().tobytes() == full[1].cpu().numpy().tobytes()
        assert torch.equal(oh, full[2])


def test_block_cyclic_pool_matches_contiguous(ams):
    """shard_block only changes placement: world=1 pools with any block size agree."""
    cfg = ams_gen.small_variant("c5", 5000, 96)
    w = ams_gen.generate_host(cfg)
    res = []
    for block in (0, 256, 7):
        with ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k, shard_block=block) as pool:
            pool.append(torch.from_numpy(w.emb).to(dev()), torch.from_numpy(w.joints).to(dev()))
            res.append([t.cpu().numpy() for t in pool.match(torch.from_numpy(w.q_emb).to(dev()),
                                                              torch.from_numpy(w.q_joints).to(dev()),
                                                              cfg.k, cfg.theta, INF)])
    for r in res[1:]:
        for a, b in zip(res[0], r):
            assert a.tobytes() == b.tobytes()
