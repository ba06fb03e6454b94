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


def _worker_bench_plumbing(rank, world, port, block, q):
    """bench.py's make_pool on CPU, without the GPU pool: every rank streams the pool
    through ams_gen.build_device_workload with the bench's chunk_needed (skip chunks this
    rank owns no row of) and keeps the rows the library's shard map assigns it."""
    dist = _init(rank, world, port)
    import dataclasses
    import hashlib
    import torch
    import ams_gen
    import paper_2508_10259_b200 as ams
    from paper_2508_10259_b200 import dist as adist
    cfg = dataclasses.replace(ams_gen.CONFIGS["c4"], M=3 * ams_gen.CHUNK_ROWS + 1234, Q=64, d=64, components=16)
    kept = {}
    state = {"off": 0, "none_owned": 0}

    def append_fn(e, j, n):
        lo = state["off"]
        for o in range(lo, lo + n):
            if ams.ams_shard_locate(cfg.M, world, block, o)[0] == rank:
                if e is None:
                    state["none_owned"] += 1        # a skipped chunk held one of our rows
                    continue
                kept[o] = hashlib.sha256(e[o - lo].view(torch.int16).numpy().tobytes() +
                                         j[o - lo].numpy().tobytes()).hexdigest()
        state["off"] += n

    need = lambda lo, hi: adist.owned_range_overlaps(cfg.M, world, block, rank, lo, hi)  # noqa: E731
    qe, qj, lab = ams_gen.build_device_workload(cfg, torch.device("cpu"), append_fn, chunk_needed=need)
    qh = hashlib.sha256(qe.view(torch.int16).numpy().tobytes() + qj.numpy().tobytes() + lab.numpy().tobytes())
    q.put((rank, kept, state["none_owned"], state["off"], qh.hexdigest()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,block", [(2, 0), (3, 0), (2, 256), (3, 256)])
def test_bench_sharded_generation_world(world, block):
    """The multi-rank data plumbing of bench.py (what the driver's SCALE run executes
    before any kernel): the union of the rows the ranks keep is the single-rank pool, row
    for row; no rank skips a chunk that holds one of its rows; queries are identical on
    every rank."""
    import dataclasses
    import hashlib
    import torch
    import ams_gen
    out = _run(_worker_bench_plumbing, world, block)
    cfg = dataclasses.replace(ams_gen.CONFIGS["c4"], M=3 * ams_gen.CHUNK_ROWS + 1234, Q=64, d=64, components=16)
    full = {}
    off = [0]

    def append_all(e, j, n):
        for r in range(n):
            full[off[0] + r] = hashlib.sha256(e[r].view(torch.int16).numpy().tobytes() + j[r].numpy().tobytes()).hexdigest()
        off[0] += n

    qe, qj, lab = ams_gen.build_device_workload(cfg, torch.device("cpu"), append_all)
    qh = hashlib.sha256(qe.view(torch.int16).numpy().tobytes() + qj.numpy().tobytes() + lab.numpy().tobytes())
    union = {}
    for rank, kept, none_owned, total, h in out:
        assert none_owned == 0 and total == cfg.M and h == qh.hexdigest(), rank
        assert not (set(union) & set(kept))
        union.update(kept)
    assert union == full
