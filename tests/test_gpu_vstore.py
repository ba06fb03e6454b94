"""GPU virtual-action store (ams_vstore_*) vs the oracle store, operation by operation."""
import numpy as np
import pytest

import oracle
from oracle.vstore import COLLISION, DEDUP, FULL, NEW, VirtualActionStore

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


def csr(actions):
    offs = np.concatenate([[0], np.cumsum([len(a) for a in actions])]).astype(np.int64)
    data = np.frombuffer(b"".join(actions), np.uint8) if offs[-1] else np.zeros(1, np.uint8)
    return np.ascontiguousarray(data), offs


def gpu_intern(ams, st, actions, ids=None, device_data=False):
    data, offs = csr(actions)
    n = len(actions)
    out_ids = torch.empty(n, dtype=torch.int64, device="cuda")
    out_st = torch.empty(n, dtype=torch.uint8, device="cuda")
    src = torch.from_numpy(data.copy()).cuda() if device_data else data
    idt = torch.from_numpy(np.array(ids, np.uint64).view(np.int64)).cuda() if ids is not None else None
    ams.ams_vstore_intern(st, src, offs, n, idt, out_ids, out_st)
    torch.cuda.synchronize()
    return out_ids.cpu().numpy().view(np.uint64), out_st.cpu().numpy()


def gpu_resolve(ams, st, ids):
    n = len(ids)
    t = torch.from_numpy(np.array(ids, np.uint64).view(np.int64)).cuda()
    off = torch.empty(n, dtype=torch.int64, device="cuda")
    ln = torch.empty(n, dtype=torch.int64, device="cuda")
    rc = torch.empty(n, dtype=torch.int64, device="cuda")
    ams.ams_vstore_resolve(st, t, n, off, ln, rc)
    torch.cuda.synchronize()
    return off.cpu().numpy(), ln.cpu().numpy(), rc.cpu().numpy()


class _DevView:
    """Zero-copy view of a raw device pointer (the store's arena) for torch.as_tensor."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def arena_slice(ams, st, off, ln):
    if ln <= 0:
        return b""
    t = torch.as_tensor(_DevView(ams.ams_vstore_arena(st) + int(off), int(ln)), device="cuda")
    return t.cpu().numpy().tobytes()


@pytest.mark.parametrize("device_data", [False, True])
def test_random_sequences_match_oracle(ams, device_data):
    rng = np.random.Generator(np.random.PCG64(21 + device_data))
    pool = [rng.integers(0, 256, rng.integers(0, 5000), dtype=np.uint8).tobytes() for _ in range(120)]
    st = ams.ams_vstore_create(0, 4096, 64 << 20, 512, 8 << 20)
    orc = VirtualActionStore()
    live = []
    for step in range(12):
        batch = [pool[i] for i in rng.integers(0, len(pool), rng.integers(1, 300))]
        ids, status = gpu_intern(ams, st, batch, device_data=device_data)
        for a, i, s in zip(batch, ids, status):
            oi, os_ = orc.intern(a)
            assert int(i) == oi
            # within one batch the GPU picks one creator among equal actions: compare counts
            assert s in (NEW, DEDUP)
        live += [int(i) for i in ids]
        # release a random subset (each at most as often as it is live)
        rng.shuffle(live)
        rel, live = live[: len(live) // 3], live[len(live) // 3:]
        if rel:
            t = torch.from_numpy(np.array(rel, np.uint64).view(np.int64)).cuda()
            rem = torch.empty(len(rel), dtype=torch.int64, device="cuda")
            ams.ams_vstore_release(st, t, len(rel), rem)
            torch.cuda.synchronize()
            exp = [orc.release(i) for i in rel]
            # final counts are order-independent; compare after the batch
        ids_all = sorted(set(live) | set(rel))
        off, ln, rc = gpu_resolve(ams, st, ids_all)
        for i, o, l, r in zip(ids_all, off, ln, rc):
            assert r == orc.refcount(i), (step, i)
            b = orc.resolve(i)
            assert (l == -1) == (b is None)
            if b is not None:
                assert l == len(b) and arena_slice(ams, st, o, l) == b
    stats = ams.ams_vstore_stats(st)
    assert stats["entries"] == len(orc.entries) and stats["total_bytes"] == orc.total_bytes
    ams.ams_vstore_destroy(st)


def test_batch_dedup_statuses_and_bytes(ams):
    a, b = b"reach-grasp-lift", b"place"
    st = ams.ams_vstore_create(0, 64, 1 << 20, 64, 1 << 20)
    ids, status = gpu_intern(ams, st, [a, b, a, a, b])
    assert ids[0] == ids[2] == ids[3] == oracle.hash_action(a) and ids[1] == ids[4] == oracle.hash_action(b)
    assert sorted(status.tolist()) == [NEW, NEW, DEDUP, DEDUP, DEDUP]
    off, ln, rc = gpu_resolve(ams, st, [int(ids[0]), int(ids[1])])
    assert rc.tolist() == [3, 2] and ln.tolist() == [len(a), len(b)]
    # bytes stored once, contiguously: the arena holds exactly len(a) + len(b) bytes
    assert ams.ams_vstore_stats(st) == {"entries": 2, "total_bytes": len(a) + len(b), "arena_used": len(a) + len(b)}
    ams.ams_vstore_destroy(st)


def test_collision_and_unknown_and_full(ams):
    st = ams.ams_vstore_create(0, 64, 100, 16, 1 << 16)
    ids, status = gpu_intern(ams, st, [b"abc"])
    forced = [int(ids[0])]
    ids2, status2 = gpu_intern(ams, st, [b"abd"], ids=forced)        # same id, different bytes
    assert status2.tolist() == [COLLISION]
    off, ln, rc = gpu_resolve(ams, st, forced)
    assert rc.tolist() == [1] and ln.tolist() == [3]
    t = torch.tensor([12345], dtype=torch.int64, device="cuda")
    rem = torch.empty(1, dtype=torch.int64, device="cuda")
    ams.ams_vstore_release(st, t, 1, rem)
    torch.cuda.synchronize()
    assert rem.item() == -1                                           # unknown id
    _, status3 = gpu_intern(ams, st, [bytes(range(200))])             # arena (100 B) too small
    assert status3.tolist() == [FULL]
    assert ams.ams_vstore_stats(st)["entries"] == 1
    ams.ams_vstore_destroy(st)


def _check_against_oracle(ams, st, orc, ids_all, tag):
    off, ln, rc = gpu_resolve(ams, st, ids_all)
    for i, o, l, r in zip(ids_all, off, ln, rc):
        assert r == orc.refcount(i), (tag, i)
        b = orc.resolve(i)
        assert (l == -1) == (b is None), (tag, i)
        if b is not None:
            assert l == len(b) and arena_slice(ams, st, o, l) == b, (tag, i)


@pytest.mark.parametrize("device_data", [False, True])
def test_churn_reclaims_arena_and_table(ams, device_data):
    """PAPER.md:583 "Any action whose reference count drops to zero is removed": 100 rounds
    of interns and releases through an arena (and table) far smaller than the bytes (and
    keys) interned over time.  Removed entries' space is reclaimed by compaction, so the
    arena top stays bounded; every live entry keeps its refcount and bytes, op by op
    against the oracle store (oracle/vstore.py)."""
    rng = np.random.Generator(np.random.PCG64(77 + device_data))
    arena = 1 << 20
    st = ams.ams_vstore_create(0, 512, arena, 128, 1 << 20)   # table: 1024 slots
    orc = VirtualActionStore()
    live = []
    interned_bytes = interned_keys = 0
    for step in range(100):
        fresh = [rng.integers(0, 256, rng.integers(0, 4000), dtype=np.uint8).tobytes()
                 for _ in range(rng.integers(1, 60))]
        again = [orc.resolve(i) for i in rng.choice(live, min(len(live), 8), replace=False)] if live else []
        batch = fresh + again
        ids, status = gpu_intern(ams, st, batch, device_data=device_data)
        assert (status != FULL).all(), step
        for a, i in zip(batch, ids):
            oi, _ = orc.intern(a)
            assert int(i) == oi
        interned_bytes += sum(len(a) for a in fresh)
        interned_keys += len(fresh)
        live += [int(i) for i in ids]
        rng.shuffle(live)
        keep = max(0, len(live) - rng.integers(len(live) // 2, len(live) + 1))
        rel, live = live[keep:], live[:keep]   # release most references: the live set stays small
        if rel:
            t = torch.from_numpy(np.array(rel, np.uint64).view(np.int64)).cuda()
            rem = torch.empty(len(rel), dtype=torch.int64, device="cuda")
            ams.ams_vstore_release(st, t, len(rel), rem)
            torch.cuda.synchronize()
            for i in rel:
                orc.release(i)
        stats = ams.ams_vstore_stats(st)
        assert stats["entries"] == len(orc.entries) and stats["total_bytes"] == orc.total_bytes, step
        assert stats["arena_used"] <= arena, step
        if step % 10 == 9:
            _check_against_oracle(ams, st, orc, sorted(set(live) | set(rel)), step)
    assert interned_bytes > 4 * arena and interned_keys > 2 * 1024   # the churn did overflow both
    ams.ams_vstore_compact(st)
    stats = ams.ams_vstore_stats(st)
    assert stats["arena_used"] == orc.total_bytes == stats["total_bytes"]   # no holes after compaction
    _check_against_oracle(ams, st, orc, sorted(set(live)), "final")
    ams.ams_vstore_destroy(st)
