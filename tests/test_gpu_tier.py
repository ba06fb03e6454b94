"""Layered storage (ams_tier_*) vs the oracle policy, op by op, with
payload round trips through HBM <-> pinned host memory."""
import numpy as np
import pytest

from oracle.tier import CapacityError, TierStore

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


@pytest.mark.parametrize("seed,fast,slow", [(0, 1 << 20, 0), (1, 300_000, 2_000_000), (2, 64_000, 0)])
def test_random_ops_match_oracle(ams, seed, fast, slow):
    rng = np.random.Generator(np.random.PCG64(seed))
    t = ams.ams_tier_create(0, fast, slow)
    orc = TierStore(fast, slow)
    payloads = {}
    next_id = 0
    for step in range(600):
        op = rng.integers(0, 4)
        if op == 0 or not orc.blobs:
            kind = int(rng.integers(0, 4))
            size = int(rng.choice([rng.integers(0, 2000), rng.integers(2000, 120_000)]))
            data = rng.integers(0, 256, size, dtype=np.uint8)
            src = torch.from_numpy(data).cuda() if rng.random() < 0.5 else data
            try:
                exp = orc.admit(next_id, kind, size)
            except CapacityError:
                with pytest.raises(ams.AmsError) as e:
                    ams.ams_tier_admit(t, next_id, kind, src, size)
                assert e.value.status == 2
            else:
                got = ams.ams_tier_admit(t, next_id, kind, src, size)
                assert got == (exp[0], [tuple(a) for a in exp[1]]), step
                payloads[next_id] = data
            next_id += 1
        elif op == 1:
            bid = int(rng.choice(list(orc.blobs)))
            orc.touch(bid)
            ams.ams_tier_touch(t, bid)
        elif op == 2:
            bid = int(rng.choice(list(orc.blobs)))
            try:
                exp = orc.fetch(bid)
            except CapacityError:
                with pytest.raises(ams.AmsError):
                    ams.ams_tier_fetch(t, bid)
            else:
                prev, dptr, acts = ams.ams_tier_fetch(t, bid)
                assert (prev, acts) == (exp[0], [tuple(a) for a in exp[1]]), step
        else:
            need = int(rng.integers(0, fast // 2 + 1))
            try:
                exp = orc.evict_until(need)
            except CapacityError:
                with pytest.raises(ams.AmsError):
                    ams.ams_tier_evict_until(t, need)
            else:
                assert ams.ams_tier_evict_until(t, need) == [tuple(a) for a in exp], step
        # state + budget invariant
        fu, su = ams.ams_tier_usage(t)
        assert fu == orc._used(0) <= fast and su == orc._used(1)
        if step % 50 == 0:
            for bid, b in orc.blobs.items():
                info = ams.ams_tier_info(t, bid)
                assert (info["tier"], info["count"], info["last"], info["size"]) == (b["tier"], b["count"], b["last"],
                                                                                    b["size"])
                if b["tier"] != 2 and b["size"] > 0:
                    out = torch.empty(b["size"], dtype=torch.uint8, device="cuda")
                    ams.ams_tier_read(t, bid, out)
                    torch.cuda.synchronize()
                    assert np.array_equal(out.cpu().numpy(), payloads[bid]), (step, bid)
    ams.ams_tier_destroy(t)


def test_vision_kv_first_and_promotion(ams):
    t = ams.ams_tier_create(0, 200 << 20)
    mk = lambda n: torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")  # noqa: E731
    a, b = mk(100 << 20), mk(100 << 20)                          # 100 MB blobs (Table 1 scale)
    assert ams.ams_tier_admit(t, 1, 2, a, a.numel())[0] == 0     # DiffusionLatent
    assert ams.ams_tier_admit(t, 2, 0, b, b.numel())[0] == 0     # VisionKV
    c = mk(50 << 20)
    placed, acts = ams.ams_tier_admit(t, 3, 1, c, c.numel())     # LlmKV
    assert acts == [(2, 2)]                                      # VisionKV dropped first
    placed, acts = ams.ams_tier_admit(t, 4, 1, mk(60 << 20), 60 << 20)
    assert acts == [(3, 1)]                                      # LlmKV (class 1) before DiffusionLatent (2)
    prev, dptr, acts = ams.ams_tier_fetch(t, 3)                  # promote 3 back; 4 is demoted for room
    assert prev == 1 and dptr and acts == [(4, 1), (3, 3)]
    out = torch.empty_like(c)
    ams.ams_tier_read(t, 3, out)
    torch.cuda.synchronize()
    assert torch.equal(out, c)                                   # bytes survived HBM -> host -> HBM
    assert ams.ams_tier_fetch(t, 2)[0] == 2                      # dropped: recompute + re-admit
    ams.ams_tier_destroy(t)
