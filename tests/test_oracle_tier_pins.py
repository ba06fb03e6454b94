"""Pins of the layered-storage oracle (oracle/tier.py) to the SPEC.md context_pool
examples and PAPER.md:592-593 ("first evict the KV Cache of vision
models"), plus the budget-safety invariant over random operation sequences."""
import numpy as np
import pytest

from oracle.tier import (DEMOTE, DIFFUSION_LATENT, DROP, DROPPED, FAST, LLM_KV, OUTPUT_EMBEDDING, PROMOTE, SLOW,
                         VISION_KV, CapacityError, TierStore)


def test_ample_budget_all_fast():                       # SPEC.md:183 [TRIVIAL]
    t = TierStore(1000)
    for i, k in enumerate([VISION_KV, LLM_KV, DIFFUSION_LATENT, OUTPUT_EMBEDDING]):
        assert t.admit(i, k, 100) == (FAST, [])


def test_vision_kv_evicted_first():
    t = TierStore(200)
    t.admit(1, DIFFUSION_LATENT, 100)
    t.admit(2, VISION_KV, 100)                          # VisionKV is the most recent, still goes first
    tier, actions = t.admit(3, OUTPUT_EMBEDDING, 50)
    assert tier == FAST and actions == [(2, DROP)]
    assert t.blobs[2]["tier"] == DROPPED and t.blobs[1]["tier"] == FAST


def test_lru_within_class():                            # SPEC.md:208 three LlmKV, distinct last_access
    t = TierStore(300)
    for i in (10, 11, 12):
        t.admit(i, LLM_KV, 100)
    t.touch(10)                                         # 11 is now the least recently used
    tier, actions = t.admit(13, LLM_KV, 100)
    assert actions == [(11, DEMOTE)] and t.blobs[11]["tier"] == SLOW


def test_touch_after_demotion_counts():
    t = TierStore(100)
    t.admit(1, LLM_KV, 100)
    t.admit(2, LLM_KV, 100)                             # demotes 1
    t.touch(1)
    t.touch(1)
    assert t.blobs[1]["tier"] == SLOW and t.blobs[1]["count"] == 2


def test_fetch_paths():
    t = TierStore(150)
    t.admit(1, VISION_KV, 100)
    t.admit(2, LLM_KV, 100)                             # drops 1 (VisionKV)
    assert t.fetch(1) == (DROPPED, [])                  # caller must recompute + re-admit
    assert t.fetch(2) == (FAST, [])
    t.admit(3, DIFFUSION_LATENT, 100)                   # demotes 2
    prev, actions = t.fetch(2)                          # promote 2: the only fast blob (3) is demoted
    assert prev == SLOW and actions == [(3, DEMOTE), (2, PROMOTE)] and t.blobs[2]["tier"] == FAST
    assert t.admit(1, VISION_KV, 40) == (FAST, [])      # re-admission of a dropped (recomputed) blob


def test_capacity_errors():
    t = TierStore(100, slow_budget=150)
    t.admit(1, LLM_KV, 100)
    t.admit(2, LLM_KV, 100)                             # 1 demoted (slow 100/150)
    with pytest.raises(CapacityError):
        t.admit(3, LLM_KV, 100)                         # demoting 2 would overflow slow
    with pytest.raises(CapacityError):
        t.admit(4, LLM_KV, 500)                         # larger than both tiers


def test_budget_safety_random():                        # SPEC.md:226 invariant
    rng = np.random.Generator(np.random.PCG64(4))
    t = TierStore(5000)
    ids = 0
    for _ in range(2000):
        op = rng.integers(0, 3)
        if op == 0 or not t.blobs:
            try:
                t.admit(ids, int(rng.integers(0, 4)), int(rng.integers(1, 2000)))
            except CapacityError:
                pass
            ids += 1
        elif op == 1:
            t.touch(int(rng.choice(list(t.blobs))))
        else:
            try:
                t.fetch(int(rng.choice(list(t.blobs))))
            except CapacityError:
                pass
        assert t._used(FAST) <= t.fast_budget
