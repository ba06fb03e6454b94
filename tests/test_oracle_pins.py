"""Pins of the CPU oracle to things other than itself.

Every test here is CPU-only.  The oracle (oracle/ams_oracle.c) is checked against:
exact-rational brute force (P1, exact fp32 fma emulation), closed forms (P2),
special cases (P3), the textbook fp64 kNN (P4), invariants (P5-P8), its own gate-
first mode (P9), the by-construction labels of the generator (P10) and the
hand-derived golden fixtures in tests/golden/ (SPEC.md examples).
"""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import ams_gen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
INF = float("inf")


def bf16(x):
    return ams_gen.f32_to_bf16_bits(np.asarray(x, np.float32))


# ----------------------------------------------------------------------------
# exact helpers (independent of the oracle)
# ----------------------------------------------------------------------------
def f32_rne(q: Fraction) -> Fraction:
    """Round an exact rational to the nearest fp32 value (ties to even)."""
    if q == 0:
        return Fraction(0)
    sign = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    # a in [2^e, 2^(e+1)); fp32 has 24 significant bits; subnormals at e < -126
    e = max(e, -126)
    ulp = Fraction(2) ** (e - 23)
    m = a / ulp
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return sign * fl * ulp


def _fr(x) -> Fraction:
    return x if isinstance(x, Fraction) else Fraction(float(x))


def fmaf_exact(a, b, c) -> Fraction:
    return f32_rne(_fr(a) * _fr(b) + _fr(c))


def rank(pairs):
    """(score, id) list -> sorted by score desc, id asc."""
    return sorted(pairs, key=lambda t: (-t[0], t[1]))


# ----------------------------------------------------------------------------
# P1: exhaustive exact pool
# ----------------------------------------------------------------------------
def _p1_pool():
    rows = np.array(list(itertools.product([-1.0, 1.0], repeat=4)), np.float32)  # 16 rows
    rng = np.random.Generator(np.random.PCG64(11))
    joints = rng.integers(-2, 3, (16, 2)).astype(np.float32)
    return rows, joints


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("gamma", [0.0, 1.0, 2.0, INF])
def test_p1_exhaustive_exact(dtype, gamma):
    rows, joints = _p1_pool()
    queries = rows.copy()
    q_joints = np.array([[0, 0], [1, -1], [2, 2], [-2, 1]] * 4, np.float32)
    emb = bf16(rows) if dtype == "bf16" else rows
    q = bf16(queries) if dtype == "bf16" else queries
    g2 = Fraction(gamma) ** 2 if gamma != INF else None
    for k in (1, 3, 5, 16, 17):
        for theta in (1.0, 0.5, 0.0, -1.0):
            res = oracle.match(emb, joints, q, q_joints, k, theta, gamma)
            for i in range(len(queries)):
                cands = []
                for j in range(16):
                    ds = sum((Fraction(float(q_joints[i, t])) - Fraction(float(joints[j, t]))) ** 2
                             for t in range(2))
                    if g2 is not None and ds > g2:
                        continue
                    dot = sum(Fraction(float(queries[i, t])) * Fraction(float(rows[j, t]))
                              for t in range(4))
                    cands.append((dot / 4, j))  # both norms are exactly 2
                exp = rank(cands)
                exp_idx = [c[1] for c in exp[:k]] + [-1] * max(0, k - len(exp))
                exp_s = [float(c[0]) for c in exp[:k]] + [-INF] * max(0, k - len(exp))
                assert res.idx[i].tolist() == exp_idx, (i, k, gamma)
                assert res.score[i].tolist() == exp_s
                exp_hit = int(len(exp) > 0 and exp[0][0] >= Fraction(theta))
                assert int(res.hit[i]) == exp_hit
                assert res.nelig[i] == len(exp)
                # (k+1)-th ranking key, used by the r = k gap rule (tests/parity.py):
                # the exact (k+1)-th enumerated score, -inf when n_elig <= k
                exp_next = float(exp[k][0]) if len(exp) > k else -INF
                assert res.next[i] == exp_next, (i, k, gamma)
                # and the full ranked keys (fp64 ranking key of each valid slot)
                assert res.key[i].tolist() == exp_s


# ----------------------------------------------------------------------------
# fp32 canonical chain vs exact fmaf emulation (brute force on tiny inputs)
# ----------------------------------------------------------------------------
def test_fp32_canonical_chain_exact_emulation():
    rng = np.random.Generator(np.random.PCG64(5))
    M, d, J, nq, k = 12, 8, 3, 4, 12
    emb = rng.standard_normal((M, d)).astype(np.float32)
    q = rng.standard_normal((nq, d)).astype(np.float32)
    joints = rng.uniform(-1, 1, (M, J)).astype(np.float32)
    qj = rng.uniform(-1, 1, (nq, J)).astype(np.float32)
    gamma = np.float32(1.1)
    res = oracle.match(emb, joints, q, qj, k, 0.3, float(gamma))

    def inv(x):
        ss = Fraction(0)
        for t in range(d):
            ss = fmaf_exact(x[t], x[t], ss)
        if ss == 0:
            return Fraction(0)
        sq = f32_rne(Fraction(math.sqrt(float(ss))))  # sqrt of an fp32 in fp64 is exact-rounded
        # fp64 sqrt is correctly rounded and fp32(fp64 sqrt) is the correctly rounded
        # fp32 sqrt (double rounding is innocuous for sqrt: 53 >= 2*24+2)
        return f32_rne(Fraction(1) / sq)

    g2 = f32_rne(Fraction(float(gamma)) * Fraction(float(gamma)))
    for i in range(nq):
        iq = inv(q[i])
        cands = []
        for j in range(M):
            ds = Fraction(0)
            for t in range(J):
                diff = f32_rne(Fraction(float(qj[i, t])) - Fraction(float(joints[j, t])))
                ds = fmaf_exact(diff, diff, ds)
            if ds > g2:
                continue
            acc = Fraction(0)
            for t in range(d):
                acc = fmaf_exact(q[i, t], emb[j, t], acc)
            s = f32_rne(f32_rne(acc * iq) * inv(emb[j]))
            cands.append((s, j))
        exp = rank(cands)
        for r in range(k):
            if r < len(exp):
                assert res.idx[i, r] == exp[r][1]
                assert Fraction(float(res.score[i, r])) == exp[r][0]
            else:
                assert res.idx[i, r] == -1


# ----------------------------------------------------------------------------
# P2: Pythagorean closed forms; norms
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_p2_pythagorean(dtype):
    rows = np.array([[3, 4, 0, 0], [4, 3, 0, 0], [0, 5, 0, 0], [0, 0, 12, 5], [5, 0, 12, 0]], np.float32)
    q = np.array([[5, 0, 0, 0], [0, 0, 5, 12]], np.float32)
    # q0 = (1,0,0,0): 3/5, 4/5, 0, 0, 5/13.  q1 = (0,0,5,12)/13: rows 0-2 orthogonal,
    # row3 (0,0,12,5)/13 -> (60+60)/169, row4 (5,0,12,0)/13 -> 60/169
    cos = np.array([[3 / 5, 4 / 5, 0, 0, 5 / 13], [0, 0, 0, 120 / 169, 60 / 169]])
    emb = bf16(rows) if dtype == "bf16" else rows
    qq = bf16(q) if dtype == "bf16" else q
    j = np.zeros((5, 1), np.float32)
    qj = np.zeros((2, 1), np.float32)
    res = oracle.match(emb, j, qq, qj, 5, 0.5, INF)
    for i in range(2):
        for r in range(5):
            jj = res.idx[i, r]
            tol = 2e-16 if dtype == "bf16" else 3 * 2.0 ** -24
            assert abs(res.key[i, r] - cos[i, jj]) <= tol, (i, r, jj)
    inv = oracle.inv_norm(emb)
    assert np.allclose(inv, [1 / 5, 1 / 5, 1 / 5, 1 / 13, 1 / 13], rtol=0, atol=1e-16 if dtype == "bf16" else 6e-8)


# ----------------------------------------------------------------------------
# P3: special cases
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_p3_special_cases(dtype):
    rows = np.array([[0, 0, 0, 0], [1, 2, 3, 4], [1, 2, 3, 4], [-1, -2, -3, -4]], np.float32)
    emb = bf16(rows) if dtype == "bf16" else rows
    q = np.array([[1, 2, 3, 4], [0, 0, 0, 0]], np.float32)
    qq = bf16(q) if dtype == "bf16" else q
    j = np.zeros((4, 2), np.float32)
    qj = np.zeros((2, 2), np.float32)
    res = oracle.match(emb, j, qq, qj, 6, 0.99, INF)
    # duplicate rows 1 and 2: the lower index first; zero row scores exactly 0 (R8)
    assert res.idx[0].tolist() == [1, 2, 0, 3, -1, -1]
    assert res.score[0, 2] == 0.0 and res.score[0, 3] <= -0.99
    assert np.all(np.isneginf(res.score[0, 4:]))
    assert res.hit[0] == 1
    # zero-norm query: every score 0 -> ranked by index, miss (0 < 0.99)
    assert res.idx[1].tolist() == [0, 1, 2, 3, -1, -1]
    assert res.score[1, :4].tolist() == [0.0] * 4 and res.hit[1] == 0
    # empty pool -> all padding, miss
    e0 = emb[:0]
    r0 = oracle.match(e0, j[:0], qq, qj, 3, -INF, INF)
    assert (r0.idx == -1).all() and (r0.hit == 0).all() and np.isneginf(r0.score).all()
    # theta = -inf: any eligible row is a hit; theta = +inf: never
    assert oracle.match(emb, j, qq, qj, 1, -INF, INF).hit.tolist() == [1, 1]
    assert oracle.match(emb, j, qq, qj, 1, INF, INF).hit.tolist() == [0, 0]


# ----------------------------------------------------------------------------
# P4: gamma = inf reduces to textbook exact cosine kNN (numpy fp64)
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_p4_textbook_knn(seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    M, d, nq, k = 300, 64, 20, 9
    # non-unit rows with varied scale: swapping inv_q / inv_e or dropping one fails
    e = (rng.standard_normal((M, d)) * rng.uniform(0.1, 10, (M, 1))).astype(np.float32)
    q = (rng.standard_normal((nq, d)) * rng.uniform(0.1, 10, (nq, 1))).astype(np.float32)
    eb, qb = bf16(e), bf16(q)
    E = ams_gen.bf16_bits_to_f32(eb).astype(np.float64)
    Qm = ams_gen.bf16_bits_to_f32(qb).astype(np.float64)
    S = (Qm / np.linalg.norm(Qm, axis=1, keepdims=True)) @ (E / np.linalg.norm(E, axis=1, keepdims=True)).T
    res = oracle.match(eb, np.zeros((M, 3), np.float32), qb, np.zeros((nq, 3), np.float32), k, 0.0, INF)
    for i in range(nq):
        full = np.lexsort((np.arange(M), -S[i]))
        order = full[:k]
        assert np.allclose(res.key[i], S[i, order], rtol=0, atol=1e-12)
        assert res.idx[i].tolist() == order.tolist()
        # the (k+1)-th key is the lexsorted (k+1)-th score (not the k-th)
        assert abs(res.next[i] - S[i, full[k]]) <= 1e-12
        assert res.next[i] <= res.key[i, k - 1]
    # fewer eligible rows than k + 1: next is -inf
    small = oracle.match(eb[:k], np.zeros((k, 3), np.float32), qb, np.zeros((nq, 3), np.float32), k, 0.0, INF)
    assert np.all(np.isneginf(small.next))
    one_more = oracle.match(eb[:k + 1], np.zeros((k + 1, 3), np.float32), qb, np.zeros((nq, 3), np.float32),
                            k, 0.0, INF)
    S1 = S[:, :k + 1]
    for i in range(nq):
        assert abs(one_more.next[i] - S1[i].min()) <= 1e-12


# ----------------------------------------------------------------------------
# P5: self-match
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_p5_self_match(dtype):
    cfg = ams_gen.small_variant("c2", 3000, 16) if dtype == "bf16" else ams_gen.CONFIGS["c1"]
    w = ams_gen.generate_host(cfg)
    pick = np.arange(0, cfg.M, max(1, cfg.M // 16))[:16]
    res = oracle.match(w.emb, w.joints, w.emb[pick], w.joints[pick], 3, 0.999, 0.3)
    tol = 1e-12 if dtype == "bf16" else 2 * 2.0 ** -23
    for n, j in enumerate(pick):
        assert res.idx[n, 0] <= j
        top = res.idx[n, 0]
        assert np.array_equal(w.emb[top], w.emb[j])
        assert abs(res.key[n, 0] - 1.0) <= tol
        assert res.hit[n] == 1


# ----------------------------------------------------------------------------
# P6: row permutation
# ----------------------------------------------------------------------------
def test_p6_row_permutation():
    w = ams_gen.generate_host(ams_gen.small_variant("c2", 2000, 24))
    base = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, 10, 0.92, INF)
    perm = np.random.Generator(np.random.PCG64(3)).permutation(2000)
    # carry the global ids: identical output
    r1 = oracle.match(w.emb[perm], w.joints[perm], w.q_emb, w.q_joints, 10, 0.92, INF, row_ids=perm)
    assert np.array_equal(r1.idx, base.idx) and np.array_equal(r1.key, base.key)
    # positional ids: indices are permuted, score multiset unchanged
    r2 = oracle.match(w.emb[perm], w.joints[perm], w.q_emb, w.q_joints, 10, 0.92, INF)
    assert np.array_equal(r2.key, base.key)
    gaps = np.diff(base.key, axis=1) != 0
    mapped = perm[r2.idx]
    for i in range(len(base.idx)):
        for r in range(10):
            left_tie = r > 0 and not gaps[i, r - 1]
            right_tie = r < 9 and not gaps[i, r]
            if not (left_tie or right_tie):
                assert mapped[i, r] == base.idx[i, r]


# ----------------------------------------------------------------------------
# P7: monotonicity in theta and gamma
# ----------------------------------------------------------------------------
def test_p7_monotonicity():
    w = ams_gen.generate_host(ams_gen.small_variant("c2", 4000, 64))
    hits = [oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, 4, th, INF).hit for th in (0.1, 0.2, 0.5, 0.95)]
    for a, b in zip(hits, hits[1:]):
        assert np.all(b <= a)
    prev = None
    for g in (0.0, 0.3, 1.0, 3.0, 10.0, INF):
        r = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, 6, 0.5, g)
        if prev is not None:
            assert np.all(r.nelig >= prev.nelig)
            assert np.all(r.key >= prev.key)
        prev = r


# ----------------------------------------------------------------------------
# P8: shard invariance (oracle side): any split + merge = unsharded, bit for bit
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("G,block", [(2, 0), (3, 0), (4, 64), (8, 256)])
def test_p8_shard_invariance(G, block):
    w = ams_gen.generate_host(ams_gen.small_variant("c2", 3001, 32))
    M = 3001
    k = 10
    base = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, k, 0.92, INF)
    ids = np.arange(M)
    B = block if block else -(-M // G)
    owner = (ids // B) % G
    keys, idxs = [], []
    for g in range(G):
        rows = ids[owner == g]
        r = oracle.match(w.emb[rows], w.joints[rows], w.q_emb, w.q_joints, k, 0.92, INF, row_ids=rows)
        keys.append(r.key)
        idxs.append(r.idx)
    m = oracle.merge(np.stack(keys), np.stack(idxs), k, 0.92)
    assert np.array_equal(m.idx, base.idx)
    assert np.array_equal(m.key, base.key)
    assert np.array_equal(m.score, base.score)
    assert np.array_equal(m.hit, base.hit)


# ----------------------------------------------------------------------------
# P9: mode A == mode B
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["c1", "c2small"])
def test_p9_mode_a_equals_b(name):
    cfg = ams_gen.CONFIGS["c1"] if name == "c1" else ams_gen.small_variant("c2", 5000, 128)
    w = ams_gen.generate_host(cfg)
    for gamma in (cfg.gamma, 2.5, INF):
        a = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma, mode="A")
        b = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, gamma, mode="B")
        for f in ("idx", "score", "hit", "key", "nelig"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f


# ----------------------------------------------------------------------------
# P10: by construction (R12-R14)
# ----------------------------------------------------------------------------
def test_p10_c1_by_construction():
    cfg = ams_gen.CONFIGS["c1"]
    w = ams_gen.generate_host(cfg)
    nd = w.labels >= 0
    assert nd.sum() == 32
    g = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, cfg.gamma)
    assert np.array_equal(g.hit.astype(bool), nd)
    assert np.array_equal(g.idx[nd, 0], w.labels[nd])
    assert (g.idx[nd, 1:] == -1).all() and (g.idx[~nd] == -1).all()
    assert np.all(np.abs(g.score[nd, 0] - 0.9988) < 2e-3)
    u = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, INF)
    assert np.array_equal(u.hit.astype(bool), nd)
    assert np.array_equal(u.idx[nd, 0], w.labels[nd])
    assert (u.idx >= 0).all()


def test_p10_c2small_by_construction():
    cfg = ams_gen.small_variant("c2", 20000, 256)
    w = ams_gen.generate_host(cfg)
    nd = w.labels >= 0
    g = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, cfg.k, cfg.theta, cfg.gamma, mode="B")
    assert np.array_equal(g.hit.astype(bool), nd)
    assert np.array_equal(g.idx[nd, 0], w.labels[nd])
    assert g.score[nd, 0].min() > 0.99 and (g.score[~nd, 0] < 0.5).all()


# ----------------------------------------------------------------------------
# golden fixtures (hand-derived from SPEC.md examples)
# ----------------------------------------------------------------------------
def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _arr(fx, key, dtype):
    a = np.array(fx[key], np.float32)
    return bf16(a) if dtype == "bf16" else a


def _f(x):
    return float(x) if not isinstance(x, str) else float(x.replace("inf", "inf"))


@pytest.mark.parametrize("name", ["spec_select_context_order.json", "spec_lookup_threshold.json"])
def test_golden_fixtures(name):
    fx = _load(name)
    assert fx["citation"]
    for dtype in ("bf16", "fp32"):
        r = oracle.match(_arr(fx, "pool_emb", dtype), np.array(fx["pool_joints"], np.float32),
                         _arr(fx, "queries_emb", dtype), np.array(fx["queries_joints"], np.float32),
                         fx["k"], fx["theta"], fx["gamma"])
        assert r.idx.tolist() == fx["expect"]["idx"]
        assert r.hit.tolist() == fx["expect"]["hit"]
        exp_s = np.array([[_f(v) for v in row] for row in fx["expect"]["score"]], np.float64)
        fin = np.isfinite(exp_s)
        assert np.all(np.isneginf(r.score[~fin]))
        assert np.allclose(r.score[fin], exp_s[fin], rtol=0, atol=max(fx["score_atol"], 1e-7))


def test_golden_gate_boundary():
    fx = _load("gate_boundary.json")
    for dtype in ("bf16", "fp32"):
        for case in fx["cases"]:
            g = _f(case["gamma"])
            r = oracle.match(_arr(fx, "pool_emb", dtype), np.array(fx["pool_joints"], np.float32),
                             _arr(fx, "queries_emb", dtype), np.array(fx["queries_joints"], np.float32),
                             fx["k"], fx["theta"], g)
            assert r.idx.tolist() == case["expect"]["idx"], (dtype, g)
            assert r.hit.tolist() == case["expect"]["hit"]
