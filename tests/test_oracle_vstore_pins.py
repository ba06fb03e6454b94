"""Pins of the virtual-action store oracle: the SPEC.md examples."""
import numpy as np

from oracle.vstore import COLLISION, DEDUP, NEW, VirtualActionStore


def test_intern_twice_dedups():          # SPEC.md:122 intern(x); intern(x) -> same id, refcount 2, stored once
    s = VirtualActionStore()
    a, st1 = s.intern(b"pick-place")
    b, st2 = s.intern(b"pick-place")
    assert a == b and (st1, st2) == (NEW, DEDUP) and s.refcount(a) == 2 and s.total_bytes == 10


def test_two_distinct():                 # SPEC.md:123 total_bytes = |x| + |y|
    s = VirtualActionStore()
    s.intern(b"x" * 7)
    s.intern(b"y" * 11)
    assert s.total_bytes == 18 and len(s.entries) == 2


def test_many_interns_of_few_distinct():  # SPEC.md:124 1000 interns of 50 distinct -> sum of the 50
    rng = np.random.Generator(np.random.PCG64(0))
    acts = [rng.integers(0, 256, rng.integers(1, 300), dtype=np.uint8).tobytes() for _ in range(50)]
    s = VirtualActionStore()
    for i in rng.integers(0, 50, 1000):
        s.intern(acts[i])
    assert s.total_bytes == sum(len(set_a) for set_a in set(acts))


def test_release_and_resolve():
    s = VirtualActionStore()
    i, _ = s.intern(b"abc")
    s.intern(b"abc")
    assert s.release(i) == 1 and s.resolve(i) == b"abc"
    assert s.release(i) == 0 and s.resolve(i) is None and s.total_bytes == 0
    assert s.release(i) == -1            # unknown id


def test_collision_changes_nothing():    # SPEC.md:119 CollisionError
    s = VirtualActionStore()
    i, _ = s.intern(b"abc")
    j, st = s.intern(b"abd", id_=i)
    assert j == i and st == COLLISION and s.resolve(i) == b"abc" and s.refcount(i) == 1
