"""Virtual-action store oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain Python, following PAPER.md:577-584 (3.2.3, "virtual action") and the SPEC.md
action_index module: ids are two-phase hashes (oracle.hash_action);
intern of identical bytes increments the reference count and stores the bytes once;
intern of different bytes under an existing id is a collision and changes nothing; a
release that brings the count to zero removes the entry; unknown ids are errors.
"""
from __future__ import annotations

from typing import Dict, List, Optional

from . import hash_action

NEW, DEDUP, COLLISION, FULL = 0, 1, 2, 3


class VirtualActionStore:
    def __init__(self):
        self.entries: Dict[int, List] = {}     # id -> [bytes, refcount]

    def intern(self, data: bytes, id_: Optional[int] = None):
        i = hash_action(data) if id_ is None else id_
        e = self.entries.get(i)
        if e is None:
            self.entries[i] = [bytes(data), 1]
            return i, NEW
        if e[0] != bytes(data):
            return i, COLLISION
        e[1] += 1
        return i, DEDUP

    def release(self, i: int) -> int:
        e = self.entries.get(i)
        if e is None:
            return -1
        e[1] -= 1
        if e[1] == 0:
            del self.entries[i]
            return 0
        return e[1]

    def resolve(self, i: int) -> Optional[bytes]:
        e = self.entries.get(i)
        return None if e is None else e[0]

    def refcount(self, i: int) -> int:
        e = self.entries.get(i)
        return 0 if e is None else e[1]

    @property
    def total_bytes(self) -> int:
        return sum(len(e[0]) for e in self.entries.values())
