"""Layered-storage / auto-eviction oracle -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

Plain Python, following PAPER.md:497-522 (3.2.2 "Layered Storage of Action Context",
Table `tab:design:cache-size`) and PAPER.md:586-594 (3.2.3 "Auto Eviction"), as
concretised by SPEC.md:158-240 (context_pool):
  * blob kinds and use classes: VisionKV -> low, LlmKV -> medium, DiffusionLatent and
    OutputEmbedding -> high (Table 1's "Use Frequency" column);
  * admit: place in the fast tier (GPU) when it fits, evicting otherwise; a blob larger
    than the fast budget goes to the slow tier (CPU); CapacityError only if it fits in
    neither;
  * touch: access_count += 1, last_access = clock, clock += 1;
  * evict_until(needed): victims in ascending P = 1000*class_rank + 1*recency_rank
    (class_rank VisionKV 0 < LlmKV 1 < DiffusionLatent = OutputEmbedding 2; recency_rank
    = rank by last_access among fast-resident blobs, 0 = least recently used), ties by
    least-recently-used then lowest blob id; VisionKV is dropped ("can be easily
    recalculated"), everything else demoted to the slow tier; stop once
    >= needed bytes are freed; CapacityError (no change) if the fast tier cannot free that
    much;
  * fetch: counts as an access; a slow blob is promoted to the fast tier (may evict); a
    dropped blob reports DROPPED and must be re-admitted by the caller after recompute.
Readings not fixed by SPEC: admission sets last_access = clock and
advances the clock; fetch of a fast blob is a touch; slow budget 0 = unbounded.
"""
from __future__ import annotations

VISION_KV, LLM_KV, DIFFUSION_LATENT, OUTPUT_EMBEDDING = 0, 1, 2, 3
CLASS_RANK = {VISION_KV: 0, LLM_KV: 1, DIFFUSION_LATENT: 2, OUTPUT_EMBEDDING: 2}
W_CLASS, W_LRU = 1000, 1
FAST, SLOW, DROPPED = 0, 1, 2
DEMOTE, DROP, PROMOTE = 1, 2, 3


class CapacityError(Exception):
    pass


class TierStore:
    def __init__(self, fast_budget: int, slow_budget: int = 0):
        self.fast_budget = fast_budget
        self.slow_budget = slow_budget
        self.clock = 0
        self.blobs = {}   # id -> dict(kind, size, tier, count, last)

    def _used(self, tier):
        return sum(b["size"] for b in self.blobs.values() if b["tier"] == tier)

    def _slow_fits(self, size):
        return self.slow_budget == 0 or self._used(SLOW) + size <= self.slow_budget

    def victims(self):
        fast = [(bid, b) for bid, b in self.blobs.items() if b["tier"] == FAST]
        by_recency = sorted(fast, key=lambda t: (t[1]["last"], t[0]))
        rank = {bid: r for r, (bid, _) in enumerate(by_recency)}
        return sorted(fast, key=lambda t: (W_CLASS * CLASS_RANK[t[1]["kind"]] + W_LRU * rank[t[0]],
                                           t[1]["last"], t[0]))

    def evict_until(self, needed: int):
        if needed <= 0:
            return []
        if self._used(FAST) < needed:
            raise CapacityError("fast tier cannot free enough")
        plan, freed = [], 0
        for bid, b in self.victims():
            if freed >= needed:
                break
            plan.append((bid, DROP if b["kind"] == VISION_KV else DEMOTE))
            freed += b["size"]
        slow_add = sum(self.blobs[bid]["size"] for bid, a in plan if a == DEMOTE)
        if not self._slow_fits(slow_add):
            raise CapacityError("slow tier full")
        for bid, a in plan:
            self.blobs[bid]["tier"] = DROPPED if a == DROP else SLOW
        return plan

    def admit(self, bid: int, kind: int, size: int):
        if bid in self.blobs and self.blobs[bid]["tier"] != DROPPED:
            raise KeyError("blob already present")
        actions = []
        if size <= self.fast_budget:
            over = self._used(FAST) + size - self.fast_budget
            actions = self.evict_until(over) if over > 0 else []
            tier = FAST
        elif self._slow_fits(size):
            tier = SLOW
        else:
            raise CapacityError("blob fits in no tier")
        self.blobs[bid] = {"kind": kind, "size": size, "tier": tier, "count": 0, "last": self.clock}
        self.clock += 1
        return tier, actions

    def touch(self, bid: int):
        b = self.blobs[bid]
        b["count"] += 1
        b["last"] = self.clock
        self.clock += 1

    def fetch(self, bid: int):
        b = self.blobs[bid]
        prev = b["tier"]
        if prev == DROPPED:
            return prev, []
        self.touch(bid)
        actions = []
        if prev == SLOW and b["size"] <= self.fast_budget:
            over = self._used(FAST) + b["size"] - self.fast_budget
            if over > 0:
                actions = self.evict_until(over)
            b["tier"] = FAST
            actions = actions + [(bid, PROMOTE)]
        return prev, actions
