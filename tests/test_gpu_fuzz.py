"""Randomized differential test of ams_match / ams_match_gate_first / ams_match_auto against
the oracle: seeded random shapes (M, d, J, nq, k), gate radii, thresholds, dtypes, kernel
policies, append chunking (host and device sources), block-cyclic shard maps on a 1-rank
NCCL communicator (the world > 1 code path), and the fused exchange on top of it -- so the
plan logic (K2 on one CTA or CTA pairs, the small-batch kernel on one CTA or CTA pairs,
narrow or wide, the gate-first variant, the fp32 exact path, the merges) is exercised in
combinations the targeted tests do not enumerate.

Inputs are drawn here (numpy PCG64): unit rows with near-duplicate queries (so hits and
filled lists occur) and fresh random ones; joints on a small lattice so exact distance ties
and gate-boundary pairs are common.  Expected values come only from oracle/.
"""
import numpy as np
import pytest

import ams_gen
import oracle
from tests.parity import check_bf16, check_exact

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
INF = float("inf")
N_CASES = int(__import__("os").environ.get("AMS_FUZZ_CASES", "72"))   # a longer sweep: AMS_FUZZ_CASES=600


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def draw_case(seed):
    rng = np.random.Generator(np.random.PCG64(10_000 + seed))
    dtype = "fp32" if rng.random() < 0.15 else "bf16"
    d = int(rng.choice([64, 128, 256, 512, 768, 1024]))
    J = int(rng.integers(1, 17))
    M = int(rng.choice([1, 7, 255, 256, 257, 1000, 3001, 9000, 20011]))
    nq = int(rng.choice([1, 2, 17, 31, 64, 65, 100, 128, 129, 150, 200, 255, 256, 300, 600]))
    k = int(rng.choice([1, 2, 5, 8, 9, 16, 17, 32, 33, 64]))
    gamma = float(rng.choice([0.0, 0.25, 0.5, 1.0, 2.0, 4.0, INF]))
    theta = float(rng.choice([-1.0, 0.0, 0.5, 0.9, 0.99]))
    policy = int(rng.choice([0, 0, 0, 1, 2, 4, 8, 12]))
    route = str(rng.choice(["dense", "dense", "gate_first", "auto"]))
    chunks = int(rng.integers(1, 4))
    host_src = bool(rng.random() < 0.3)
    shard = str(rng.choice(["local", "local", "collective", "peer"]))
    block = int(rng.choice([0, 256, 1000]))
    # rows: unit vectors; joints on a 0.25-rad lattice (exact ties, gate-boundary pairs)
    e = rng.standard_normal((M, d)).astype(np.float32)
    e /= np.linalg.norm(e, axis=1, keepdims=True)
    pj = (rng.integers(-8, 9, (M, J)) * 0.25).astype(np.float32)
    if M > 3:
        e[1] = e[0]          # exact duplicate rows: the lower index first
        pj[1] = pj[0]
    src = rng.integers(0, M, nq)
    near = rng.random(nq) < 0.5
    q = rng.standard_normal((nq, d)).astype(np.float32)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    noisy = e[src] + (0.05 / np.sqrt(d)) * rng.standard_normal((nq, d)).astype(np.float32)
    noisy /= np.linalg.norm(noisy, axis=1, keepdims=True)
    q[near] = noisy[near]
    qj = (rng.integers(-8, 9, (nq, J)) * 0.25).astype(np.float32)
    qj[near] = pj[src[near]] + (rng.integers(-1, 2, (int(near.sum()), J)) * 0.25).astype(np.float32)
    if dtype == "bf16":
        e, q = ams_gen.f32_to_bf16_bits(e), ams_gen.f32_to_bf16_bits(q)
    return dict(dtype=dtype, d=d, J=J, M=M, nq=nq, k=k, gamma=gamma, theta=theta, policy=policy, route=route,
                chunks=chunks, host_src=host_src, shard=shard, block=block, e=e, pj=pj, q=q, qj=qj)


@pytest.mark.parametrize("seed", range(N_CASES))
def test_fuzz_against_oracle(ams, seed):
    c = draw_case(seed)
    nid = ams.ams_get_nccl_unique_id() if c["shard"] != "local" else None
    pool = ams.Pool(c["d"], c["J"], c["M"], c["nq"], c["k"], dtype=c["dtype"], nccl_id=nid, shard_block=c["block"])
    try:
        if c["shard"] == "peer" and c["dtype"] == "bf16":
            ams.ams_pool_enable_peer_exchange(pool.handle)
        ams.ams_pool_set_kernel_policy(pool.handle, c["policy"])
        bounds = np.unique(np.linspace(0, c["M"], c["chunks"] + 1).astype(int))
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            e, pj = c["e"][lo:hi], c["pj"][lo:hi]
            first = pool.append(e if c["host_src"] else T(e), pj if c["host_src"] else T(pj), hi - lo)
            assert first == lo
        qv = T(c["q"]).view(torch.bfloat16) if c["dtype"] == "bf16" else T(c["q"])
        gf = {"dense": False, "gate_first": True, "auto": "auto"}[c["route"]]
        out = [t.cpu().numpy() for t in pool.match(qv, T(c["qj"]), c["k"], c["theta"], c["gamma"], gate_first=gf)]
        torch.cuda.synchronize()
        assert ams.ams_pool_status(pool.handle) == 0
    finally:
        pool.close()
    orc = oracle.match(c["e"], c["pj"], c["q"], c["qj"], c["k"], c["theta"], c["gamma"])
    ctx = {x: c[x] for x in ("dtype", "d", "J", "M", "nq", "k", "gamma", "theta", "policy", "route", "chunks",
                             "host_src", "shard", "block")}
    if c["dtype"] == "fp32":
        check_exact(*out, orc)
    else:
        try:
            check_bf16(*out, orc, c["theta"])
        except AssertionError as err:
            raise AssertionError(f"{ctx}: {err}") from None
