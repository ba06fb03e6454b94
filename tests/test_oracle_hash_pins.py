"""Pins of the oracle's two-phase action hash (Alg. 1 `lst:impl:index`,
PAPER.md:538-574; SPEC.md:103-111 concretisation B=257, M=2^61-1, s=4096).

Pinned against: the SPEC examples (empty -> 0; shorter than s -> h_1), hand closed
forms, an independent power-sum formula in Python big integers (sum_j b_j B^(n-1-j)
mod M per segment, sum_i h_i B^(k-1-i) mod M -- not the oracle's Horner loop), and
segment-boundary cases.
"""
import numpy as np
import pytest

import oracle

B, M, S = 257, (1 << 61) - 1, 4096


def power_sum(xs, base=B):
    n = len(xs)
    return sum(int(x) * pow(base, n - 1 - j, M) for j, x in enumerate(xs)) % M


def two_phase_power_sum(data: bytes, s=S):
    if not data:
        return 0
    hs = [power_sum(data[o:o + s]) for o in range(0, len(data), s)]
    return power_sum(hs)


def test_spec_examples():
    # SPEC.md:108 "empty input -> 0 (zero segments, empty fold)"
    assert oracle.hash_action(b"") == 0
    # SPEC.md:109 "input shorter than s -> H_final = h_1"
    x = bytes(range(200))
    assert oracle.hash_action(x) == oracle.hash_segment(x)


def test_closed_forms():
    assert oracle.hash_action(b"\x05") == 5
    assert oracle.hash_action(b"\x01\x02") == 257 + 2
    assert oracle.hash_action(b"\x01\x00\x00") == 257 * 257
    assert oracle.hash_action(b"\xff" * 3) == 255 * (257 ** 2 + 257 + 1)
    # two full segments of s=2: H = h1*B + h2
    assert oracle.hash_action(b"\x01\x02\x03\x04", s=2) == ((1 * 257 + 2) * 257 + (3 * 257 + 4)) % M


@pytest.mark.parametrize("n,s", [(1, 4096), (4095, 4096), (4096, 4096), (4097, 4096), (10240, 4096),
                                 (100000, 4096), (777, 16), (1000, 1), (65537, 8192)])
def test_power_sum_form(n, s):
    rng = np.random.Generator(np.random.PCG64(n * 31 + s))
    data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
    assert oracle.hash_action(data, s=s) == two_phase_power_sum(data, s)


def test_modulus_wraps():
    data = b"\xff" * 50000   # many wraps of 2^61 - 1
    assert oracle.hash_action(data) == two_phase_power_sum(data)
    assert oracle.hash_action(data) < M


def test_one_byte_difference_changes_hash():
    # SPEC.md:110 "two 10 KiB inputs differing in one byte -> different hashes"
    rng = np.random.Generator(np.random.PCG64(3))
    a = bytearray(rng.integers(0, 256, 10240, dtype=np.uint8).tobytes())
    b = bytearray(a)
    b[5000] ^= 0x40
    assert oracle.hash_action(bytes(a)) != oracle.hash_action(bytes(b))


def test_batch_form_matches_single():
    rng = np.random.Generator(np.random.PCG64(8))
    lens = rng.integers(0, 9000, 40)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    data = rng.integers(0, 256, int(offs[-1]), dtype=np.uint8)
    out = oracle.hash_actions(data, offs)
    for i in range(40):
        assert int(out[i]) == oracle.hash_action(data[offs[i]:offs[i + 1]].tobytes())
