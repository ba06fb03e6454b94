"""Fused NVLink shard exchange: the producer/consumer kernels behind
ams_pool_enable_peer_exchange, run for G virtual ranks on one GPU by
ams_exchange_selftest (every consumer is enqueued after the producers it waits for, so
no kernel waits on a concurrently running one).

Each virtual rank's result of each round must equal the oracle's k-way merge
(oracle.merge, "similar context" = best scores; the ordering/tie rule is
DESIGN.md reading R6) of that round's G lists, bit for bit -- every round with fresh
data, so a consumer that read a stale parity slot or an old epoch fails.
"""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


def ranked_lists(rng, rounds, G, nq, k):
    """[rounds, G, nq, k] lists ordered by (score desc, id asc) with ties across ranks,
    ragged (-inf, -1) tails and ids unique per (round, query)."""
    s = rng.choice(np.linspace(-1, 1, 7).astype(np.float32), (rounds, G, nq, k))
    ids = np.empty((rounds, G, nq, k), np.int64)
    for r in range(rounds):
        for i in range(nq):
            ids[r, :, i, :] = rng.permutation(G * k * 3)[: G * k].reshape(G, k) + r * 1_000_003
    for r in range(rounds):
        for g in range(G):
            for i in range(nq):
                o = np.lexsort((ids[r, g, i], -s[r, g, i]))
                s[r, g, i], ids[r, g, i] = s[r, g, i][o], ids[r, g, i][o]
                cut = rng.integers(0, k + 1)
                s[r, g, i, cut:] = -np.inf
                ids[r, g, i, cut:] = -1
    return np.ascontiguousarray(s), np.ascontiguousarray(ids)


@pytest.mark.parametrize("G,nq,k,rounds", [(1, 5, 4, 2), (2, 257, 16, 3), (3, 100, 5, 4), (8, 130, 32, 3),
                                           (4, 33, 64, 2), (8, 1, 1, 5), (5, 4097, 8, 2)])
def test_exchange_matches_oracle_merge(ams, G, nq, k, rounds):
    rng = np.random.Generator(np.random.PCG64(G * 1000 + k))
    s, ids = ranked_lists(rng, rounds, G, nq, k)
    th = 0.3
    dev = torch.device("cuda", 0)
    out_s = torch.empty(rounds, G, nq, k, dtype=torch.float32, device=dev)
    out_i = torch.empty(rounds, G, nq, k, dtype=torch.int64, device=dev)
    out_h = torch.empty(rounds, G, nq, dtype=torch.uint8, device=dev)
    ams.ams_exchange_selftest(G, nq, k, rounds, th, torch.from_numpy(s).to(dev), torch.from_numpy(ids).to(dev),
                              out_s, out_i, out_h)
    os_, oi, oh = out_s.cpu().numpy(), out_i.cpu().numpy(), out_h.cpu().numpy()
    for r in range(rounds):
        orc = oracle.merge(s[r].astype(np.float64), ids[r], k, th)
        for g in range(G):   # every rank holds the same merged answer
            assert np.array_equal(oi[r, g], orc.idx), (r, g)
            assert os_[r, g].tobytes() == orc.score.astype(np.float32).tobytes(), (r, g)
            assert np.array_equal(oh[r, g], orc.hit), (r, g)


@pytest.mark.parametrize("G,nq,k,rounds", [(2, 65, 8, 4), (8, 130, 16, 3), (3, 1, 1, 5)])
def test_exchange_late_consumer(ams, G, nq, k, rounds):
    """A consumer that runs after its peers already raised their flags for the NEXT epoch
    (the order a descheduled host thread produces) must still merge the right epoch's
    lists (wait is flag >= epoch; the parity slot is intact).  With an equality wait
    this order times out and the call returns AMS_ERR_NCCL."""
    rng = np.random.Generator(np.random.PCG64(G * 77 + k))
    s, ids = ranked_lists(rng, rounds, G, nq, k)
    dev = torch.device("cuda", 0)
    out_s = torch.empty(rounds, G, nq, k, dtype=torch.float32, device=dev)
    out_i = torch.empty(rounds, G, nq, k, dtype=torch.int64, device=dev)
    out_h = torch.empty(rounds, G, nq, dtype=torch.uint8, device=dev)
    ams.ams_exchange_selftest(G, nq, k, rounds, 0.3, torch.from_numpy(s).to(dev), torch.from_numpy(ids).to(dev),
                              out_s, out_i, out_h, flags=ams.AMS_SELFTEST_LATE_CONSUMER)
    oi, oh = out_i.cpu().numpy(), out_h.cpu().numpy()
    for r in range(rounds):
        orc = oracle.merge(s[r].astype(np.float64), ids[r], k, 0.3)
        for g in range(G):
            assert np.array_equal(oi[r, g], orc.idx), (r, g)
            assert np.array_equal(oh[r, g], orc.hit), (r, g)


def test_exchange_timeout_reports_error(ams):
    """A peer that never delivers: the bounded wait ends (20 ms in the self-test), the
    outputs of the lost round are padding, earlier rounds are intact, and the call
    returns AMS_ERR_NCCL instead of hanging the GPU."""
    G, nq, k, rounds = 3, 40, 8, 2
    rng = np.random.Generator(np.random.PCG64(5))
    s, ids = ranked_lists(rng, rounds, G, nq, k)
    dev = torch.device("cuda", 0)
    out_s = torch.zeros(rounds, G, nq, k, dtype=torch.float32, device=dev)
    out_i = torch.zeros(rounds, G, nq, k, dtype=torch.int64, device=dev)
    out_h = torch.ones(rounds, G, nq, dtype=torch.uint8, device=dev)
    with pytest.raises(ams.AmsError) as e:
        ams.ams_exchange_selftest(G, nq, k, rounds, 0.3, torch.from_numpy(s).to(dev), torch.from_numpy(ids).to(dev),
                                  out_s, out_i, out_h, flags=ams.AMS_SELFTEST_DROP_LAST)
    assert e.value.status == 5
    torch.cuda.synchronize()   # the device is still healthy
    oi, os_, oh = out_i.cpu().numpy(), out_s.cpu().numpy(), out_h.cpu().numpy()
    orc = oracle.merge(s[0].astype(np.float64), ids[0], k, 0.3)
    for g in range(G):
        assert np.array_equal(oi[0, g], orc.idx)
    for g in range(G - 1):   # the consumers that waited for the dropped producer
        assert (oi[1, g] == -1).all() and np.isneginf(os_[1, g]).all() and (oh[1, g] == 0).all()


def test_exchange_rejects_bad_arguments(ams):
    dev = torch.device("cuda", 0)
    x = torch.zeros(16, device=dev)
    i = torch.zeros(16, dtype=torch.int64, device=dev)
    h = torch.zeros(16, dtype=torch.uint8, device=dev)
    for G, nq, k, rounds, fl in [(0, 1, 1, 1, 0), (9, 1, 1, 1, 0), (1, 0, 1, 1, 0), (1, 1, 65, 1, 0),
                                 (1, 1, 1, 0, 0), (2, 1, 1, 1, 4), (1, 1, 1, 1, 1)]:
        with pytest.raises(ams.AmsError) as e:
            ams.ams_exchange_selftest(G, nq, k, rounds, 0.5, x, i, x, i, h, flags=fl)
        assert e.value.status == 1


def test_enable_peer_exchange_needs_peers(ams):
    pool = ams.ams_pool_create(64, 4, 1024, 8, 8)
    with pytest.raises(ams.AmsError) as e:
        ams.ams_pool_enable_peer_exchange(pool)      # world 1: nothing to exchange
    assert e.value.status == 6
    ams.ams_pool_destroy(pool)
