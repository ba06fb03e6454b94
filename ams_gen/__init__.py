"""Seeded synthetic inputs for action-context matching (AMS, arXiv 2508.10259).

This module is the ONLY code shared between the oracle tests and the CUDA path.
It draws pools and queries; it holds none of the method's arithmetic (no norms
used for scoring, no dot products, no gate, no top-k, no threshold).

Recipe (SURVEY.md 8(d) and readings R12-R17):

* The pool stands in for "data from the robot's joints and the output embedding
  obtained from the final inference" (3.2.1): one embedding row of
  width d plus a J-DoF joint vector per context.
* ``unit(x)``: fp32 L2 normalisation of a generator draw, then (bf16 configs)
  round-to-nearest-even to bf16 storage.  This is input shaping, not scoring.
* Embeddings: C1 i.i.d. N(0, I); C2-C5 a Gaussian mixture whose component means
  are unit(N(0, I)) and whose per-coordinate within-component spread is 0.1 (R13).
* Joints: i.i.d. U[-pi, pi]^J (R14).
* Queries: a fraction are near-duplicates of pool rows drawn WITHOUT replacement
  (embedding noise N(0, (0.05/sqrt(d))^2) per coordinate on the stored row, then
  unit (R12); joint noise N(0, 0.02^2)); the rest are fresh (C1: unit(N(0,I)),
  mixture configs: fresh mixture samples), with fresh uniform joints.  Queries are
  shuffled by a seeded permutation; ``labels[i]`` is the near-duplicate source row
  or -1.
* Small configs are drawn with numpy PCG64 on the host; the large ones (C3-C5)
  with torch Philox on the GPU in fixed 65,536-row chunks seeded by
  (seed, chunk), so the pool is identical for every GPU count and shard map.
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import Optional

import numpy as np

PI = math.pi
CHUNK_ROWS = 65536


# ----------------------------------------------------------------------------
# bf16 storage helpers (bit-level, RNE). Storage encoding, not method arithmetic.
# ----------------------------------------------------------------------------
def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (round to nearest, ties to even); returns uint16 bits."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    out = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """Exact decode of bf16 bits to fp32."""
    b = np.ascontiguousarray(b, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32)


def _unit_np(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.float32)
    n = np.sqrt(np.sum(x * x, axis=1, keepdims=True, dtype=np.float32))
    n[n == 0] = 1.0
    return (x / n).astype(np.float32)


def sha256_of(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


# ----------------------------------------------------------------------------
# Config table (BASELINE.json configs[0..4] = C1..C5)
# ----------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    seed: int
    M: int
    d: int
    J: int
    Q: int
    near_dup_frac: float
    k: int
    theta: float
    gamma: float
    dtype: str              # "bf16" | "fp32"
    components: int         # 0 -> i.i.d. N(0, I) embeddings (C1)
    device_gen: bool        # True -> torch CUDA chunked generator


CONFIGS = {
    # BASELINE.json configs[0]
    "c1": Config("c1", 1, 1024, 512, 7, 64, 0.5, 5, 0.9, 0.3, "fp32", 0, False),
    # configs[1]
    "c2": Config("c2", 2, 100_000, 768, 7, 4096, 0.5, 10, 0.92, 0.3, "bf16", 256, False),
    # configs[2]
    "c3": Config("c3", 3, 1 << 20, 1024, 14, 16384, 0.25, 16, 0.9, 0.3, "bf16", 1024, True),
    # north_star "64-query scan" on C3's pool (R17)
    "c3scan": Config("c3scan", 3, 1 << 20, 1024, 14, 64, 0.25, 16, 0.9, 0.3, "bf16", 1024, True),
    # configs[3]
    "c4": Config("c4", 4, 1 << 24, 1024, 7, 8192, 0.25, 32, 0.9, 0.3, "bf16", 1024, True),
    # configs[4] (initial pool; streaming appends drawn by stream_rows())
    "c5": Config("c5", 5, 1 << 22, 4096, 7, 256, 0.5, 8, 0.9, 0.3, "bf16", 1024, True),
}


def small_variant(name: str, M: int, Q: int, seed_offset: int = 100) -> Config:
    """Scaled-down twin of a config (same d, J, k, theta, gamma, dtype, mixture)
    drawn on the host; used for oracle-complete parity at tile-spanning sizes."""
    c = CONFIGS[name]
    return dataclasses.replace(c, name=f"{name}_M{M}_Q{Q}", seed=c.seed + seed_offset,
                               M=M, Q=Q, device_gen=False,
                               components=min(c.components, max(M // 8, 1)) if c.components else 0)


@dataclasses.dataclass
class Workload:
    cfg: Config
    emb: np.ndarray          # [M, d] uint16 (bf16 bits) or float32
    joints: np.ndarray       # [M, J] float32
    q_emb: np.ndarray        # [Q, d] same dtype as emb
    q_joints: np.ndarray     # [Q, J] float32
    labels: np.ndarray       # [Q] int64 near-duplicate source row, -1 for fresh

    def sha256(self) -> str:
        return sha256_of(self.emb, self.joints, self.q_emb, self.q_joints)


# ----------------------------------------------------------------------------
# Host (numpy PCG64) generator
# ----------------------------------------------------------------------------
def _store(x_f32: np.ndarray, dtype: str) -> np.ndarray:
    return f32_to_bf16_bits(x_f32) if dtype == "bf16" else x_f32.astype(np.float32)


def _decode(x: np.ndarray, dtype: str) -> np.ndarray:
    return bf16_bits_to_f32(x) if dtype == "bf16" else x.astype(np.float32)


def generate_host(cfg: Config) -> Workload:
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    M, d, J, Q = cfg.M, cfg.d, cfg.J, cfg.Q
    if cfg.components:
        means = _unit_np(rng.standard_normal((cfg.components, d), dtype=np.float32))
        comp = rng.integers(0, cfg.components, M)
        x = means[comp] + np.float32(0.1) * rng.standard_normal((M, d), dtype=np.float32)
    else:
        means = None
        x = rng.standard_normal((M, d), dtype=np.float32)
    emb = _store(_unit_np(x), cfg.dtype)
    joints = rng.uniform(-PI, PI, (M, J)).astype(np.float32)

    n_nd = int(round(Q * cfg.near_dup_frac))
    n_nd = min(n_nd, M)
    src = rng.choice(M, n_nd, replace=False).astype(np.int64)
    sigma = np.float32(0.05 / math.sqrt(d))
    q_nd = _decode(emb[src], cfg.dtype) + sigma * rng.standard_normal((n_nd, d), dtype=np.float32)
    qj_nd = joints[src] + np.float32(0.02) * rng.standard_normal((n_nd, J), dtype=np.float32)
    n_fr = Q - n_nd
    if means is not None:
        comp_q = rng.integers(0, cfg.components, n_fr)
        q_fr = means[comp_q] + np.float32(0.1) * rng.standard_normal((n_fr, d), dtype=np.float32)
    else:
        q_fr = rng.standard_normal((n_fr, d), dtype=np.float32)
    qj_fr = rng.uniform(-PI, PI, (n_fr, J)).astype(np.float32)

    q = np.concatenate([_unit_np(q_nd), _unit_np(q_fr)], axis=0)
    qj = np.concatenate([qj_nd, qj_fr], axis=0).astype(np.float32)
    labels = np.concatenate([src, -np.ones(n_fr, np.int64)])
    perm = rng.permutation(Q)
    return Workload(cfg, emb, joints, _store(q[perm], cfg.dtype),
                    np.ascontiguousarray(qj[perm]), labels[perm])


# ----------------------------------------------------------------------------
# Device (torch Philox, chunked) generator for the large configs
# ----------------------------------------------------------------------------
def _torch():
    import torch  # local import: the host generator must not need torch
    return torch


def _unit_t(x):
    torch = _torch()
    n = torch.linalg.vector_norm(x, dim=1, keepdim=True)
    return x / torch.where(n == 0, torch.ones_like(n), n)


def device_means(cfg: Config, device):
    torch = _torch()
    g = torch.Generator(device=device).manual_seed(cfg.seed * 1_000_003 + 7)
    return _unit_t(torch.randn(cfg.components, cfg.d, generator=g, device=device))


def device_pool_chunk(cfg: Config, chunk: int, means, device, rows: Optional[int] = None):
    """Rows [chunk*CHUNK_ROWS, ...) of the pool: (emb bf16 [n,d], joints f32 [n,J])."""
    torch = _torch()
    n = rows if rows is not None else min(CHUNK_ROWS, cfg.M - chunk * CHUNK_ROWS)
    g = torch.Generator(device=device).manual_seed(cfg.seed * 1_000_003 + 1000 + chunk)
    comp = torch.randint(0, cfg.components, (n,), generator=g, device=device)
    x = means[comp] + 0.1 * torch.randn(n, cfg.d, generator=g, device=device)
    emb = _unit_t(x).to(torch.bfloat16)
    joints = (torch.rand(n, cfg.J, generator=g, device=device) * (2 * PI) - PI).float()
    return emb, joints


def device_pool(cfg: Config, device, out_emb=None, out_joints=None):
    """Whole pool on `device` (bf16 [M,d], f32 [M,J]); optionally into given buffers."""
    torch = _torch()
    means = device_means(cfg, device)
    if out_emb is None:
        out_emb = torch.empty(cfg.M, cfg.d, dtype=torch.bfloat16, device=device)
        out_joints = torch.empty(cfg.M, cfg.J, dtype=torch.float32, device=device)
    nchunks = (cfg.M + CHUNK_ROWS - 1) // CHUNK_ROWS
    for c in range(nchunks):
        e, j = device_pool_chunk(cfg, c, means, device)
        out_emb[c * CHUNK_ROWS: c * CHUNK_ROWS + e.shape[0]] = e
        out_joints[c * CHUNK_ROWS: c * CHUNK_ROWS + e.shape[0]] = j
    return out_emb, out_joints


def device_queries(cfg: Config, pool_emb, pool_joints, device, Q: Optional[int] = None,
                   salt: int = 0, src_lo: int = 0, src_hi: Optional[int] = None):
    """Queries for a device-generated pool: (q bf16 [Q,d], qj f32 [Q,J], labels i64 [Q]).

    Near-duplicate sources are drawn without replacement from rows [src_lo, src_hi).
    """
    torch = _torch()
    Q = cfg.Q if Q is None else Q
    src_hi = pool_emb.shape[0] if src_hi is None else src_hi
    g = torch.Generator(device=device).manual_seed(cfg.seed * 1_000_003 + 999 + salt * 7919)
    n_nd = int(round(Q * cfg.near_dup_frac))
    n_nd = min(n_nd, src_hi - src_lo)
    if src_hi - src_lo <= 4 * n_nd + 1024:
        src = torch.randperm(src_hi - src_lo, generator=g, device=device)[:n_nd] + src_lo
    else:  # draw without replacement by rejection of duplicates (pools up to 2^24)
        cand = torch.randint(src_lo, src_hi, (2 * n_nd + 64,), generator=g, device=device)
        src = torch.unique(cand)
        src = src[torch.randperm(src.numel(), generator=g, device=device)][:n_nd]
        assert src.numel() == n_nd
    src = src.to(torch.int64)
    sigma = 0.05 / math.sqrt(cfg.d)
    q_nd = pool_emb[src].float() + sigma * torch.randn(n_nd, cfg.d, generator=g, device=device)
    qj_nd = pool_joints[src] + 0.02 * torch.randn(n_nd, cfg.J, generator=g, device=device)
    n_fr = Q - n_nd
    means = device_means(cfg, device)
    comp = torch.randint(0, cfg.components, (n_fr,), generator=g, device=device)
    q_fr = means[comp] + 0.1 * torch.randn(n_fr, cfg.d, generator=g, device=device)
    qj_fr = torch.rand(n_fr, cfg.J, generator=g, device=device) * (2 * PI) - PI
    q = torch.cat([_unit_t(q_nd), _unit_t(q_fr)]).to(torch.bfloat16)
    qj = torch.cat([qj_nd, qj_fr]).float()
    labels = torch.cat([src, torch.full((n_fr,), -1, dtype=torch.int64, device=device)])
    perm = torch.randperm(Q, generator=g, device=device)
    return q[perm].contiguous(), qj[perm].contiguous(), labels[perm].contiguous()


def stream_rows(cfg: Config, step: int, n: int, device):
    """C5 streaming: the n new mixture rows appended at simulated step `step`."""
    torch = _torch()
    means = device_means(cfg, device)
    g = torch.Generator(device=device).manual_seed(cfg.seed * 1_000_003 + 5_000_000 + step)
    comp = torch.randint(0, cfg.components, (n,), generator=g, device=device)
    x = means[comp] + 0.1 * torch.randn(n, cfg.d, generator=g, device=device)
    emb = _unit_t(x).to(torch.bfloat16)
    joints = (torch.rand(n, cfg.J, generator=g, device=device) * (2 * PI) - PI).float()
    return emb, joints


def batch_sizes(total: int, seed: int):
    """C5: seeded batch sizes ~ log-uniform{1..256}, truncated to the remainder."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    left = total
    while left > 0:
        b = int(min(left, max(1, round(math.exp(rng.uniform(0.0, math.log(256.0)))))))
        out.append(b)
        left -= b
    return out


def build_device_workload(cfg: Config, device, append_fn, Q: Optional[int] = None, salt: int = 0,
                          chunk_needed=None, host_copy: bool = False):
    """Stream the pool of a device-generated config through ``append_fn(emb, joints)``
    chunk by chunk (never holding the whole pool), then draw the queries.

    ``chunk_needed(lo, hi) -> bool`` may skip generating chunks whose rows the caller
    ignores (a rank that owns none of them); append_fn then receives ``None`` for that
    chunk's arrays and must still account for ``hi - lo`` rows.  Near-duplicate source
    rows are always regenerated.  Returns (q bf16 [Q,d], qj f32 [Q,J], labels i64 [Q]) on
    `device`, plus the host copy of the pool (emb uint16 bits, joints) if host_copy.
    """
    torch = _torch()
    Q = cfg.Q if Q is None else Q
    g = torch.Generator(device="cpu").manual_seed(cfg.seed * 1_000_003 + 999 + salt * 7919)
    n_nd = min(int(round(Q * cfg.near_dup_frac)), cfg.M)
    src = torch.randperm(cfg.M, generator=g)[:n_nd] if cfg.M <= (1 << 24) else \
        torch.unique(torch.randint(0, cfg.M, (2 * n_nd + 64,), generator=g))[:n_nd]
    src = src.to(torch.int64)
    order = torch.argsort(src)
    src_sorted = src[order]
    means = device_means(cfg, device)
    src_emb = torch.empty(n_nd, cfg.d, dtype=torch.bfloat16, device=device)
    src_j = torch.empty(n_nd, cfg.J, dtype=torch.float32, device=device)
    host_e = host_j = None
    if host_copy:
        host_e = np.empty((cfg.M, cfg.d), np.uint16)
        host_j = np.empty((cfg.M, cfg.J), np.float32)
    nchunks = (cfg.M + CHUNK_ROWS - 1) // CHUNK_ROWS
    for c in range(nchunks):
        lo = c * CHUNK_ROWS
        hi = min(cfg.M, lo + CHUNK_ROWS)
        a = int(torch.searchsorted(src_sorted, lo))
        b = int(torch.searchsorted(src_sorted, hi))
        need = chunk_needed is None or chunk_needed(lo, hi)
        if need or b > a or host_copy:
            e, j = device_pool_chunk(cfg, c, means, device)
            if b > a:
                rows = (src_sorted[a:b] - lo).to(device)
                src_emb[a:b] = e[rows]
                src_j[a:b] = j[rows]
            if host_copy:
                host_e[lo:hi] = e.view(torch.int16).cpu().numpy().view(np.uint16)
                host_j[lo:hi] = j.cpu().numpy()
            append_fn(e if need else None, j if need else None, hi - lo)
        else:
            append_fn(None, None, hi - lo)
    # undo the sort: sources in draw order
    inv = torch.empty_like(order)
    inv[order] = torch.arange(n_nd)
    src_emb = src_emb[inv.to(device)]
    src_j = src_j[inv.to(device)]
    gq = torch.Generator(device=device).manual_seed(cfg.seed * 1_000_003 + 4242 + salt * 7919)
    sigma = 0.05 / math.sqrt(cfg.d)
    q_nd = src_emb.float() + sigma * torch.randn(n_nd, cfg.d, generator=gq, device=device)
    qj_nd = src_j + 0.02 * torch.randn(n_nd, cfg.J, generator=gq, device=device)
    n_fr = Q - n_nd
    comp = torch.randint(0, cfg.components, (n_fr,), generator=gq, device=device)
    q_fr = means[comp] + 0.1 * torch.randn(n_fr, cfg.d, generator=gq, device=device)
    qj_fr = torch.rand(n_fr, cfg.J, generator=gq, device=device) * (2 * PI) - PI
    q = torch.cat([_unit_t(q_nd), _unit_t(q_fr)]).to(torch.bfloat16)
    qj = torch.cat([qj_nd, qj_fr]).float()
    labels = torch.cat([src.to(device), torch.full((n_fr,), -1, dtype=torch.int64, device=device)])
    perm = torch.randperm(Q, generator=gq, device=device)
    out = (q[perm].contiguous(), qj[perm].contiguous(), labels[perm].contiguous())
    if host_copy:
        return out + (host_e, host_j)
    return out
