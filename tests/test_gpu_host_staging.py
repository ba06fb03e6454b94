"""Host-sourced appends larger than the pool's host-staging buffer (a fixed 64 MiB
budget, allocated on the first host append): the chunked staging loop of
ams_pool_append runs several times, with a ragged last chunk.  The pool must equal the
one built from device buffers, byte for byte in every output, and match the oracle."""
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


def test_host_append_spans_several_staging_chunks(ams):
    cfg = ams_gen.small_variant("c3", 70001, 96)          # d = 1024 bf16, J = 14
    w = ams_gen.generate_host(cfg)
    row = 2 * cfg.d + 4 * cfg.J
    stage_rows = (64 << 20) // row
    assert cfg.M > 2 * stage_rows                            # >= 3 chunks, the last one ragged
    dev = torch.device("cuda", 0)
    outs = []
    for host in (True, False):
        with ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k) as pool:
            if host:
                first = pool.append(np.ascontiguousarray(w.emb), np.ascontiguousarray(w.joints), cfg.M)
            else:
                first = pool.append(torch.from_numpy(w.emb).to(dev), torch.from_numpy(w.joints).to(dev), cfg.M)
            assert first == 0 and pool.size == cfg.M
            for gamma in (cfg.gamma, INF):
                outs.append([t.cpu().numpy() for t in pool.match(torch.from_numpy(w.q_emb).to(dev),
                                                                 torch.from_numpy(w.q_joints).to(dev),
                                                                 cfg.k, cfg.theta, gamma)])
    for a, b in zip(outs[:2], outs[2:]):
        for x, y in zip(a, b):
            assert x.tobytes() == y.tobytes()
    for gamma, o in zip((cfg.gamma, INF), outs[:2]):
        orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma, mode="B")
        check_bf16(*o, orc, cfg.theta)


def test_host_append_in_pieces_across_chunk_boundaries(ams):
    """Several host appends whose sizes straddle the staging chunk size."""
    cfg = ams_gen.small_variant("c5", 20011, 40)            # d = 4096: 8,164 rows per 64 MiB chunk
    w = ams_gen.generate_host(cfg)
    dev = torch.device("cuda", 0)
    with ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k) as pool:
        off = 0
        for n in (1, 8179, 8181, 3650):
            assert pool.append(np.ascontiguousarray(w.emb[off:off + n]), np.ascontiguousarray(w.joints[off:off + n]),
                               n) == off
            off += n
        assert off == cfg.M == pool.size
        o = [t.cpu().numpy() for t in pool.match(torch.from_numpy(w.q_emb).to(dev),
                                                 torch.from_numpy(w.q_joints).to(dev), cfg.k, cfg.theta, INF)]
    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, INF)
    check_bf16(*o, orc, cfg.theta)
