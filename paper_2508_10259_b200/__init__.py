"""B200-native action-context matching (AMS, arXiv 2508.10259) -- Python binding.

A thin ctypes layer over ``libams.so`` (include/ams.h).  Functions carry the C ABI
names and only marshal arguments: every step of the path runs in the CUDA kernels
of the library.  There is no CPU fallback: importing this package without the built
library raises, and every call that fails raises ``AmsError``.

Buffers may be passed as torch tensors (host or CUDA), numpy arrays (host) or raw
integer pointers.  Streams are torch.cuda.Stream objects, raw ``cudaStream_t``
integers, or None (the current torch stream when torch is importable, else the
legacy default stream).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libams.so")

ABI_VERSION = 2   # include/ams.h AMS_ABI_VERSION this binding marshals for
AMS_OK = 0
AMS_DTYPE_BF16 = 0
AMS_DTYPE_FP32 = 1
STATUS = {0: "AMS_OK", 1: "AMS_ERR_INVALID_ARGUMENT", 2: "AMS_ERR_CAPACITY", 3: "AMS_ERR_OUT_OF_MEMORY",
          4: "AMS_ERR_CUDA", 5: "AMS_ERR_NCCL", 6: "AMS_ERR_UNSUPPORTED", 7: "AMS_ERR_INTERNAL"}

# Every symbol include/ams.h declares (tests check the library exports all of them).
EXPORTS = ("ams_get_nccl_unique_id", "ams_pool_create", "ams_pool_append", "ams_match", "ams_match_gate_first",
           "ams_match_auto", "ams_pool_last_route",
           "ams_merge_topk", "ams_pool_enable_peer_exchange", "ams_exchange_selftest",
           "ams_pool_status", "ams_build_id", "ams_pool_size",
           "ams_pool_destroy", "ams_status_string", "ams_pool_set_profiling", "ams_pool_read_profile",
           "ams_pool_launch_count", "ams_pool_last_plan", "ams_pool_set_kernel_policy", "ams_shard_locate", "ams_shard_capacity",
           "ams_abi_version", "ams_hasher_create", "ams_hash_actions", "ams_hasher_last_stats", "ams_hasher_destroy",
           "ams_vstore_create", "ams_vstore_intern", "ams_vstore_release", "ams_vstore_resolve",
           "ams_vstore_arena", "ams_vstore_stats", "ams_vstore_compact", "ams_vstore_destroy", "ams_tier_create", "ams_tier_admit",
           "ams_tier_touch", "ams_tier_evict_until", "ams_tier_fetch", "ams_tier_info", "ams_tier_usage",
           "ams_tier_read", "ams_tier_destroy")


class AmsError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what} failed: {STATUS.get(status, status)}")
        self.status = status


class ams_pool_config_t(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("joint_dim", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("capacity", ctypes.c_int64), ("max_queries", ctypes.c_int32), ("max_k", ctypes.c_int32),
                ("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p), ("shard_block", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2508_10259_b200/build.py` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    V, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "ams_get_nccl_unique_id": [V],
        "ams_pool_create": [ctypes.POINTER(ams_pool_config_t), ctypes.POINTER(V)],
        "ams_pool_append": [V, V, V, I64, ctypes.POINTER(I64), V],
        "ams_match": [V, V, V, I32, I32, ctypes.c_float, ctypes.c_float, V, V, V, V],
        "ams_match_gate_first": [V, V, V, I32, I32, ctypes.c_float, ctypes.c_float, V, V, V, V],
        "ams_match_auto": [V, V, V, I32, I32, ctypes.c_float, ctypes.c_float, V, V, V, V],
        "ams_pool_last_route": [V, ctypes.POINTER(I32), ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)],
        "ams_merge_topk": [V, V, I32, I32, I32, I32, ctypes.c_float, V, V, V, V],
        "ams_pool_enable_peer_exchange": [V],
        "ams_exchange_selftest": [I32, I32, I32, I32, ctypes.c_float, V, V, V, V, V, I32, V],
        "ams_pool_status": [V],
        "ams_pool_size": [V, ctypes.POINTER(I64)],
        "ams_pool_destroy": [V],
        "ams_pool_set_profiling": [V, I32],
        "ams_pool_set_kernel_policy": [V, I32],
        "ams_pool_read_profile": [V, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64)],
        "ams_pool_launch_count": [V, ctypes.POINTER(I64)],
        "ams_pool_last_plan": [V, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I32),
                               ctypes.POINTER(I32)],
        "ams_shard_locate": [I64, I32, I64, I64, ctypes.POINTER(I32), ctypes.POINTER(I64)],
        "ams_shard_capacity": [I64, I32, I64, I32, ctypes.POINTER(I64)],
        "ams_hasher_create": [I32, I64, I64, I64, ctypes.POINTER(V)],
        "ams_hash_actions": [V, V, V, I32, V, V],
        "ams_hasher_destroy": [V],
        "ams_hasher_last_stats": [V, ctypes.POINTER(I64), ctypes.POINTER(I64)],
        "ams_vstore_create": [I32, I64, I64, I32, I64, ctypes.POINTER(V)],
        "ams_vstore_intern": [V, V, V, I32, V, V, V, V],
        "ams_vstore_release": [V, V, I32, V, V],
        "ams_vstore_resolve": [V, V, I32, V, V, V, V],
        "ams_vstore_arena": [V, ctypes.POINTER(V)],
        "ams_vstore_stats": [V, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)],
        "ams_vstore_destroy": [V],
        "ams_vstore_compact": [V, V],
        "ams_tier_create": [I32, I64, I64, ctypes.POINTER(V)],
        "ams_tier_admit": [V, I64, I32, V, I64, ctypes.POINTER(I32), V, V, I32, ctypes.POINTER(I32), V],
        "ams_tier_touch": [V, I64],
        "ams_tier_evict_until": [V, I64, V, V, I32, ctypes.POINTER(I32), V],
        "ams_tier_fetch": [V, I64, ctypes.POINTER(I32), ctypes.POINTER(V), V, V, I32, ctypes.POINTER(I32), V],
        "ams_tier_info": [V, I64, ctypes.POINTER(I32), ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)],
        "ams_tier_usage": [V, ctypes.POINTER(I64), ctypes.POINTER(I64)],
        "ams_tier_read": [V, I64, V, V],
        "ams_tier_destroy": [V],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.ams_status_string.argtypes = [ctypes.c_int]
    L.ams_status_string.restype = ctypes.c_char_p
    L.ams_abi_version.argtypes = []
    L.ams_abi_version.restype = ctypes.c_int32
    L.ams_build_id.argtypes = []
    L.ams_build_id.restype = ctypes.c_char_p
    return L


lib = _load()
if lib.ams_abi_version() != ABI_VERSION:
    raise ImportError(f"{LIB_PATH} has ABI {lib.ams_abi_version()}, this binding needs {ABI_VERSION}: rebuild it")


def _check(st: int, what: str):
    if st != AMS_OK:
        raise AmsError(st, what)


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):          # torch.Tensor
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    if hasattr(x, "ctypes"):            # numpy.ndarray
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    raise TypeError(f"cannot take a pointer of {type(x)}")


def _stream(s) -> Optional[int]:
    if s is None:
        try:
            import torch
            if torch.cuda.is_available() and torch.cuda.is_initialized():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


# ----------------------------------------------------------------------------- C ABI
def ams_abi_version() -> int:
    return int(lib.ams_abi_version())


def ams_build_id() -> str:
    return lib.ams_build_id().decode()


def ams_status_string(st: int) -> str:
    return lib.ams_status_string(st).decode()


def ams_get_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.ams_get_nccl_unique_id(buf), "ams_get_nccl_unique_id")
    return buf.raw


def ams_pool_create(dim: int, joint_dim: int, capacity: int, max_queries: int, max_k: int,
                    dtype: int = AMS_DTYPE_BF16, device: int = 0, rank: int = 0, world: int = 1,
                    nccl_id: Optional[bytes] = None, shard_block: int = 0) -> int:
    cfg = ams_pool_config_t(dim, joint_dim, dtype, capacity, max_queries, max_k, device, rank, world, None,
                            shard_block)
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        cfg.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
    out = ctypes.c_void_p()
    _check(lib.ams_pool_create(ctypes.byref(cfg), ctypes.byref(out)), "ams_pool_create")
    return out.value


def ams_pool_append(pool: int, emb, joints, n: int, stream=None) -> int:
    first = ctypes.c_int64(-1)
    _check(lib.ams_pool_append(pool, _ptr(emb), _ptr(joints), n, ctypes.byref(first), _stream(stream)),
           "ams_pool_append")
    return first.value


def ams_match(pool: int, q_emb, q_joints, nq: int, k: int, threshold: float, gate_radius: float,
              out_index, out_score, out_hit, stream=None) -> None:
    _check(lib.ams_match(pool, _ptr(q_emb), _ptr(q_joints), nq, k, threshold, gate_radius, _ptr(out_index),
                         _ptr(out_score), _ptr(out_hit), _stream(stream)), "ams_match")


def ams_match_gate_first(pool: int, q_emb, q_joints, nq: int, k: int, threshold: float, gate_radius: float,
                         out_index, out_score, out_hit, stream=None) -> None:
    _check(lib.ams_match_gate_first(pool, _ptr(q_emb), _ptr(q_joints), nq, k, threshold, gate_radius,
                                    _ptr(out_index), _ptr(out_score), _ptr(out_hit), _stream(stream)),
           "ams_match_gate_first")


def ams_match_auto(pool: int, q_emb, q_joints, nq: int, k: int, threshold: float, gate_radius: float,
                   out_index, out_score, out_hit, stream=None) -> None:
    _check(lib.ams_match_auto(pool, _ptr(q_emb), _ptr(q_joints), nq, k, threshold, gate_radius, _ptr(out_index),
                              _ptr(out_score), _ptr(out_hit), _stream(stream)), "ams_match_auto")


def ams_pool_last_route(pool: int):
    r = ctypes.c_int32()
    e, md, mg = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _check(lib.ams_pool_last_route(pool, ctypes.byref(r), ctypes.byref(e), ctypes.byref(md), ctypes.byref(mg)),
           "ams_pool_last_route")
    return {"route": {-1: None, 0: "dense", 1: "gate_first"}[r.value], "est_eligible_per_query": e.value,
            "est_ms_dense": md.value, "est_ms_gate_first": mg.value}


def ams_merge_topk(in_score, in_index, G: int, nq: int, kin: int, k: int, threshold: float, out_index,
                   out_score, out_hit, stream=None) -> None:
    _check(lib.ams_merge_topk(_ptr(in_score), _ptr(in_index), G, nq, kin, k, threshold, _ptr(out_index),
                              _ptr(out_score), _ptr(out_hit), _stream(stream)), "ams_merge_topk")


def ams_pool_enable_peer_exchange(pool: int) -> None:
    _check(lib.ams_pool_enable_peer_exchange(pool), "ams_pool_enable_peer_exchange")


AMS_SELFTEST_LATE_CONSUMER = 1
AMS_SELFTEST_DROP_LAST = 2


def ams_exchange_selftest(G: int, nq: int, k: int, rounds: int, threshold: float, in_score, in_index, out_score,
                          out_index, out_hit, flags: int = 0, stream=None) -> None:
    _check(lib.ams_exchange_selftest(G, nq, k, rounds, threshold, _ptr(in_score), _ptr(in_index), _ptr(out_score),
                                     _ptr(out_index), _ptr(out_hit), int(flags), _stream(stream)),
           "ams_exchange_selftest")


def ams_pool_status(pool: int) -> int:
    """Sticky status without a sync (AMS_ERR_NCCL after a peer-exchange timeout); returns the code."""
    return int(lib.ams_pool_status(pool))


def ams_pool_size(pool: int) -> int:
    n = ctypes.c_int64()
    _check(lib.ams_pool_size(pool, ctypes.byref(n)), "ams_pool_size")
    return n.value


def ams_pool_destroy(pool: int) -> None:
    _check(lib.ams_pool_destroy(pool), "ams_pool_destroy")


def ams_pool_set_profiling(pool: int, enable: bool) -> None:
    _check(lib.ams_pool_set_profiling(pool, 1 if enable else 0), "ams_pool_set_profiling")


def ams_pool_set_kernel_policy(pool: int, policy: int) -> None:
    """Bit mask, 0 = default.  Bit 0: no small-batch kernel (nq <= 128 uses the
    128-query-tile kernel).  Bit 1: 4-CTA clusters of two CTA pairs sharing multicast
    pool rows (opt-in; plan id 5).  Bit 2: wide small-batch CTA pairs (two tiles per
    pipeline stage instead of one; opt-in).  Bit 3: ungated 129-256-query batches on the
    small-batch CTA pairs (default: the 256-query-tile kernel)."""
    _check(lib.ams_pool_set_kernel_policy(pool, int(policy)), "ams_pool_set_kernel_policy")


def ams_pool_read_profile(pool: int):
    ms = ctypes.c_double()
    n = ctypes.c_int64()
    _check(lib.ams_pool_read_profile(pool, ctypes.byref(ms), ctypes.byref(n)), "ams_pool_read_profile")
    return ms.value, n.value


def ams_pool_launch_count(pool: int) -> int:
    n = ctypes.c_int64()
    _check(lib.ams_pool_launch_count(pool, ctypes.byref(n)), "ams_pool_launch_count")
    return n.value


def ams_pool_last_plan(pool: int):
    v = [ctypes.c_int32() for _ in range(4)]
    _check(lib.ams_pool_last_plan(pool, *[ctypes.byref(x) for x in v]), "ams_pool_last_plan")
    return {"splits": v[0].value, "partials": v[1].value, "grid": v[2].value, "kernel_id": v[3].value}


def ams_shard_locate(capacity: int, world: int, shard_block: int, global_index: int):
    o, l = ctypes.c_int32(), ctypes.c_int64()
    _check(lib.ams_shard_locate(capacity, world, shard_block, global_index, ctypes.byref(o), ctypes.byref(l)),
           "ams_shard_locate")
    return o.value, l.value


def ams_shard_capacity(capacity: int, world: int, shard_block: int, rank: int) -> int:
    n = ctypes.c_int64()
    _check(lib.ams_shard_capacity(capacity, world, shard_block, rank, ctypes.byref(n)), "ams_shard_capacity")
    return n.value


def ams_hasher_create(device: int, max_inputs: int, max_bytes: int, segment_size: int = 4096) -> int:
    out = ctypes.c_void_p()
    _check(lib.ams_hasher_create(device, max_inputs, max_bytes, segment_size, ctypes.byref(out)), "ams_hasher_create")
    return out.value


def ams_hash_actions(hasher: int, data, offsets, n_inputs: int, out_hash, stream=None) -> None:
    """offsets: host int64 array [n_inputs + 1]; data host or device; out_hash device u64."""
    import numpy as np
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    _check(lib.ams_hash_actions(hasher, _ptr(data), off.ctypes.data, n_inputs, _ptr(out_hash), _stream(stream)),
           "ams_hash_actions")


def ams_hasher_last_stats(hasher: int):
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.ams_hasher_last_stats(hasher, ctypes.byref(a), ctypes.byref(b)), "ams_hasher_last_stats")
    return {"segments": a.value, "tc_segments": b.value}


def ams_hasher_destroy(hasher: int) -> None:
    _check(lib.ams_hasher_destroy(hasher), "ams_hasher_destroy")


def ams_vstore_create(device: int, max_actions: int, arena_bytes: int, max_batch: int, max_batch_bytes: int) -> int:
    out = ctypes.c_void_p()
    _check(lib.ams_vstore_create(device, max_actions, arena_bytes, max_batch, max_batch_bytes, ctypes.byref(out)),
           "ams_vstore_create")
    return out.value


def ams_vstore_intern(store: int, data, offsets, n: int, ids_in, out_ids, out_status, stream=None) -> None:
    import numpy as np
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    _check(lib.ams_vstore_intern(store, _ptr(data), off.ctypes.data, n, _ptr(ids_in), _ptr(out_ids),
                                 _ptr(out_status), _stream(stream)), "ams_vstore_intern")


def ams_vstore_release(store: int, ids, n: int, out_remaining, stream=None) -> None:
    _check(lib.ams_vstore_release(store, _ptr(ids), n, _ptr(out_remaining), _stream(stream)), "ams_vstore_release")


def ams_vstore_resolve(store: int, ids, n: int, out_offset, out_len, out_refcount=None, stream=None) -> None:
    _check(lib.ams_vstore_resolve(store, _ptr(ids), n, _ptr(out_offset), _ptr(out_len), _ptr(out_refcount),
                                  _stream(stream)), "ams_vstore_resolve")


def ams_vstore_arena(store: int) -> int:
    p = ctypes.c_void_p()
    _check(lib.ams_vstore_arena(store, ctypes.byref(p)), "ams_vstore_arena")
    return p.value


def ams_vstore_stats(store: int):
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib.ams_vstore_stats(store, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), "ams_vstore_stats")
    return {"entries": a.value, "total_bytes": b.value, "arena_used": c.value}


def ams_vstore_compact(store: int, stream=None) -> None:
    _check(lib.ams_vstore_compact(store, _stream(stream)), "ams_vstore_compact")


def ams_vstore_destroy(store: int) -> None:
    _check(lib.ams_vstore_destroy(store), "ams_vstore_destroy")


def _acts(max_acts=64):
    import numpy as np
    return np.zeros(max_acts, np.int64), np.zeros(max_acts, np.int32), ctypes.c_int32(0)


def _acts_list(ids, kinds, n):
    m = min(n.value, len(ids))
    return [(int(ids[i]), int(kinds[i])) for i in range(m)]


def ams_tier_create(device: int, fast_budget: int, slow_budget: int = 0) -> int:
    out = ctypes.c_void_p()
    _check(lib.ams_tier_create(device, fast_budget, slow_budget, ctypes.byref(out)), "ams_tier_create")
    return out.value


def ams_tier_admit(tier: int, blob_id: int, kind: int, payload, size: int, stream=None):
    """Returns (placed_tier, [(blob_id, action), ...])."""
    ids, kinds, n = _acts()
    placed = ctypes.c_int32(-1)
    _check(lib.ams_tier_admit(tier, blob_id, kind, _ptr(payload), size, ctypes.byref(placed), ids.ctypes.data,
                              kinds.ctypes.data, len(ids), ctypes.byref(n), _stream(stream)), "ams_tier_admit")
    return placed.value, _acts_list(ids, kinds, n)


def ams_tier_touch(tier: int, blob_id: int) -> None:
    _check(lib.ams_tier_touch(tier, blob_id), "ams_tier_touch")


def ams_tier_evict_until(tier: int, needed: int, stream=None):
    ids, kinds, n = _acts()
    _check(lib.ams_tier_evict_until(tier, needed, ids.ctypes.data, kinds.ctypes.data, len(ids), ctypes.byref(n),
                                    _stream(stream)), "ams_tier_evict_until")
    return _acts_list(ids, kinds, n)


def ams_tier_fetch(tier: int, blob_id: int, stream=None):
    """Returns (prev_tier, device_ptr or None, [(blob_id, action), ...])."""
    ids, kinds, n = _acts()
    prev = ctypes.c_int32(-1)
    dp = ctypes.c_void_p()
    _check(lib.ams_tier_fetch(tier, blob_id, ctypes.byref(prev), ctypes.byref(dp), ids.ctypes.data,
                              kinds.ctypes.data, len(ids), ctypes.byref(n), _stream(stream)), "ams_tier_fetch")
    return prev.value, dp.value, _acts_list(ids, kinds, n)


def ams_tier_info(tier: int, blob_id: int):
    t, c, l, s = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib.ams_tier_info(tier, blob_id, ctypes.byref(t), ctypes.byref(c), ctypes.byref(l), ctypes.byref(s)),
           "ams_tier_info")
    return {"tier": t.value, "count": c.value, "last": l.value, "size": s.value}


def ams_tier_usage(tier: int):
    f, s = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.ams_tier_usage(tier, ctypes.byref(f), ctypes.byref(s)), "ams_tier_usage")
    return f.value, s.value


def ams_tier_read(tier: int, blob_id: int, dst, stream=None) -> None:
    _check(lib.ams_tier_read(tier, blob_id, _ptr(dst), _stream(stream)), "ams_tier_read")


def ams_tier_destroy(tier: int) -> None:
    _check(lib.ams_tier_destroy(tier), "ams_tier_destroy")


# ----------------------------------------------------------------------------- convenience
class Pool:
    """RAII handle over an ams pool with torch CUDA output allocation (marshalling only)."""

    def __init__(self, dim, joint_dim, capacity, max_queries, max_k, dtype="bf16", device=0, rank=0, world=1,
                 nccl_id=None, shard_block=0):
        self.dim, self.joint_dim, self.device = dim, joint_dim, device
        self.dtype = AMS_DTYPE_BF16 if dtype in ("bf16", AMS_DTYPE_BF16) else AMS_DTYPE_FP32
        self.handle = ams_pool_create(dim, joint_dim, capacity, max_queries, max_k, self.dtype, device, rank,
                                      world, nccl_id, shard_block)

    def append(self, emb, joints, n=None, stream=None) -> int:
        n = emb.shape[0] if n is None else n
        return ams_pool_append(self.handle, emb, joints, n, stream)

    def match(self, q_emb, q_joints, k, threshold, gate_radius, out=None, stream=None, gate_first=False):
        import torch
        nq = q_emb.shape[0]
        if out is None:
            dev = torch.device("cuda", self.device)
            out = (torch.empty(nq, k, dtype=torch.int64, device=dev),
                   torch.empty(nq, k, dtype=torch.float32, device=dev),
                   torch.empty(nq, dtype=torch.uint8, device=dev))
        fn = ams_match_auto if gate_first == "auto" else ams_match_gate_first if gate_first else ams_match
        fn(self.handle, q_emb, q_joints, nq, k, threshold, gate_radius, out[0], out[1], out[2], stream)
        return out

    @property
    def size(self) -> int:
        return ams_pool_size(self.handle)

    def close(self):
        if self.handle:
            h, self.handle = self.handle, None
            ams_pool_destroy(h)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
