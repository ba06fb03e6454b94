"""World-size-2 tests of the multi-GPU host path on CPU (torch.distributed / gloo).

The GPU exchange (NCCL all-gather inside ams_match) cannot run in this container;
these tests cover what surrounds it:
  * the NCCL unique-id bootstrap (rank 0 draws it through the C ABI; the bytes are
    broadcast over the process group) -- paper_2508_10259_b200.dist.bootstrap_nccl_id;
  * the sharded protocol itself on the oracle side: every rank keeps the rows the
    library's shard map assigns it, computes its shard's exact top-k, the lists are
    all-gathered and merged, and the result equals the unsharded oracle bit for bit
    (pin P8 across real processes).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _worker_bootstrap(rank, world, port, q):
    dist = _init(rank, world, port)
    from paper_2508_10259_b200.dist import bootstrap_nccl_id
    nid = bootstrap_nccl_id()
    gathered = [None] * world
    dist.all_gather_object(gathered, nid)
    q.put((rank, nid, gathered))
    dist.destroy_process_group()


def _worker_sharded(rank, world, port, block, q):
    dist = _init(rank, world, port)
    import torch
    import ams_gen
    import oracle
    import paper_2508_10259_b200 as ams
    cfg = ams_gen.small_variant("c4", 2501, 48)
    w = ams_gen.generate_host(cfg)
    owner = np.array([ams.ams_shard_locate(cfg.M, world, block, o)[0] for o in range(cfg.M)])
    rows = np.nonzero(owner == rank)[0]
    res = []
    for gamma in (cfg.gamma, float("inf"), 2.0):
        r = oracle.match(w.emb[rows], w.joints[rows], w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma, row_ids=rows)
        keys = [torch.zeros_like(torch.from_numpy(r.key)) for _ in range(world)]
        ids = [torch.zeros_like(torch.from_numpy(r.idx)) for _ in range(world)]
        dist.all_gather(keys, torch.from_numpy(r.key))
        dist.all_gather(ids, torch.from_numpy(r.idx))
        m = oracle.merge(np.stack([k.numpy() for k in keys]), np.stack([i.numpy() for i in ids]), cfg.k, cfg.theta)
        full = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma)
        res.append(bool(np.array_equal(m.idx, full.idx) and np.array_equal(m.key, full.key)
                        and np.array_equal(m.hit, full.hit) and np.array_equal(m.score, full.score)))
    q.put((rank, res, int(rows.size)))
    dist.destroy_process_group()


def _run(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def test_nccl_id_bootstrap_world2():
    out = _run(_worker_bootstrap, 2)
    ids = [o[1] for o in out]
    assert all(isinstance(i, bytes) and len(i) == 128 for i in ids)
    assert ids[0] == ids[1]
    assert out[0][2] == out[1][2]


@pytest.mark.parametrize("block", [0, 256])
def test_sharded_protocol_world2_equals_unsharded(block):
    out = _run(_worker_sharded, 2, block)
    assert sum(o[2] for o in out) == 2501
    for rank, res, _ in out:
        assert all(res), (rank, res)
