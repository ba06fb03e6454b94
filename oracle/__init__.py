"""CPU oracle for AMS action-context matching -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2508_10259_b200``) never imports it, and it imports nothing from the
product path.  The arithmetic lives in ``ams_oracle.c`` (plain C, fp64 for bf16
inputs, canonical fp32 for fp32 inputs), which cites the passages it follows.

Pins (tests/test_oracle_pins.py): exhaustive exact pool P1 against an
exact-rational brute force, Pythagorean closed forms P2, special cases P3, the
textbook kNN reduction P4 (gamma = inf vs numpy fp64), invariants P5-P8, Mode A =
Mode B P9 and the by-construction labels P10.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ams_oracle.c")
_LIB = os.path.join(_HERE, "libams_oracle.so")
_lock = threading.Lock()
_lib = None

BF16, FP32 = 0, 1
CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            L.oracle_match.restype = ctypes.c_int
            L.oracle_match.argtypes = [ctypes.c_int32, P, P, P, ctypes.c_int64, ctypes.c_int32,
                                       ctypes.c_int32, P, P, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_float, ctypes.c_float, ctypes.c_int32,
                                       ctypes.c_int32, P, P, P, P, P, P]
            L.oracle_merge.restype = ctypes.c_int
            L.oracle_merge.argtypes = [P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_float, P, P, P, P]
            L.oracle_inv_norm_bf16.argtypes = [P, ctypes.c_int64, ctypes.c_int32, P]
            L.oracle_inv_norm_f32.argtypes = [P, ctypes.c_int64, ctypes.c_int32, P]
            L.oracle_gate_ds.restype = ctypes.c_float
            L.oracle_gate_ds.argtypes = [P, P, ctypes.c_int32]
            L.oracle_gate_g2.restype = ctypes.c_float
            L.oracle_gate_g2.argtypes = [ctypes.c_float]
            L.oracle_max_threads.restype = ctypes.c_int
            L.oracle_hash_action.restype = ctypes.c_uint64
            L.oracle_hash_action.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64]
            L.oracle_hash_segment.restype = ctypes.c_uint64
            L.oracle_hash_segment.argtypes = [P, ctypes.c_int64, ctypes.c_uint64]
            L.oracle_hash_actions.restype = None
            L.oracle_hash_actions.argtypes = [P, P, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, P]
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Result:
    """Oracle output for nq queries: idx [nq,k] int64 (-1 pad), score [nq,k] fp32
    (-inf pad), hit [nq] u8, key [nq,k] fp64 ranking key, next [nq] (k+1)-th key,
    nelig [nq] eligible-row count."""

    def __init__(self, nq, k):
        self.idx = np.empty((nq, k), np.int64)
        self.score = np.empty((nq, k), np.float32)
        self.hit = np.empty(nq, np.uint8)
        self.key = np.empty((nq, k), np.float64)
        self.next = np.empty(nq, np.float64)
        self.nelig = np.empty(nq, np.int64)


def _dtype_code(emb: np.ndarray) -> int:
    if emb.dtype == np.uint16:
        return BF16
    if emb.dtype == np.float32:
        return FP32
    raise TypeError(f"embedding dtype must be uint16 (bf16 bits) or float32, got {emb.dtype}")


def match(emb, joints, q_emb, q_joints, k, theta, gamma, mode="A", row_ids=None, threads=0):
    """Oracle matcher (ams_oracle.c:oracle_match).  emb: [M,d] uint16 bf16 bits or
    float32; joints [M,J] float32; queries likewise.  mode "A" brute force, "B" gate first."""
    emb = np.ascontiguousarray(emb)
    q_emb = np.ascontiguousarray(q_emb, dtype=emb.dtype)
    joints = np.ascontiguousarray(joints, dtype=np.float32)
    q_joints = np.ascontiguousarray(q_joints, dtype=np.float32)
    M, d = emb.shape
    nq = q_emb.shape[0]
    J = joints.shape[1]
    assert q_emb.shape[1] == d and q_joints.shape == (nq, J) and joints.shape[0] == M
    rid = None
    if row_ids is not None:
        rid = np.ascontiguousarray(row_ids, dtype=np.int64)
        assert rid.shape == (M,)
    res = Result(nq, k)
    rc = lib().oracle_match(_dtype_code(emb), _p(emb), _p(joints), _p(rid) if rid is not None else None,
                            M, d, J, _p(q_emb), _p(q_joints), nq, k, float(theta), float(gamma),
                            1 if mode == "B" else 0, int(threads), _p(res.idx), _p(res.score),
                            _p(res.hit), _p(res.key), _p(res.next), _p(res.nelig))
    if rc != 0:
        raise RuntimeError("oracle_match failed")
    return res


def merge(keys, ids, k, theta):
    """Merge G ranked lists [G,nq,kin] by (key desc, id asc) into top-k."""
    keys = np.ascontiguousarray(keys, dtype=np.float64)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    G, nq, kin = keys.shape
    res = Result(nq, k)
    rc = lib().oracle_merge(_p(keys), _p(ids), G, nq, kin, k, float(theta), _p(res.idx),
                            _p(res.score), _p(res.hit), _p(res.key))
    if rc != 0:
        raise RuntimeError("oracle_merge failed")
    return res


def inv_norm(x):
    """Step 1: inverse L2 norms (fp64 for bf16 bits, canonical fp32 for float32)."""
    x = np.ascontiguousarray(x)
    n, d = x.shape
    if x.dtype == np.uint16:
        out = np.empty(n, np.float64)
        lib().oracle_inv_norm_bf16(_p(x), n, d, _p(out))
    else:
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(n, np.float32)
        lib().oracle_inv_norm_f32(_p(x), n, d, _p(out))
    return out


def gate_ds(r, p):
    r = np.ascontiguousarray(r, dtype=np.float32)
    p = np.ascontiguousarray(p, dtype=np.float32)
    return float(lib().oracle_gate_ds(_p(r), _p(p), r.shape[0]))


def gate_g2(gamma):
    return float(lib().oracle_gate_g2(float(gamma)))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


HASH_B = 257
HASH_M = (1 << 61) - 1
HASH_S = 4096


def hash_action(data: bytes, s: int = HASH_S, B: int = HASH_B) -> int:
    """Two-phase action hash (Alg. 1): ams_oracle.c."""
    buf = np.frombuffer(bytes(data), dtype=np.uint8) if len(data) else np.zeros(1, np.uint8)
    return int(lib().oracle_hash_action(_p(buf), len(data), s, B))


def hash_segment(data: bytes, B: int = HASH_B) -> int:
    buf = np.frombuffer(bytes(data), dtype=np.uint8) if len(data) else np.zeros(1, np.uint8)
    return int(lib().oracle_hash_segment(_p(buf), len(data), B))


def hash_actions(data: np.ndarray, offsets: np.ndarray, s: int = HASH_S, B: int = HASH_B) -> np.ndarray:
    """Batch form over a CSR byte buffer: input i is data[offsets[i]:offsets[i+1]]."""
    data = np.ascontiguousarray(data, dtype=np.uint8)
    if data.size == 0:
        data = np.zeros(1, np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    out = np.empty(len(offsets) - 1, np.uint64)
    lib().oracle_hash_actions(_p(data), _p(offsets), len(offsets) - 1, s, B, _p(out))
    return out
