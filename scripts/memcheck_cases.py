"""Small cases of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):  compute-sanitizer --tool memcheck python scripts/memcheck_cases.py"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import ams_gen, oracle
import paper_2508_10259_b200 as ams
from tests.parity import check_bf16, check_exact
torch.cuda.set_device(0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
INF = float("inf")
# fp32 exact + bf16 (CTA-pair and single-CTA) + gate-first, ragged sizes
for name, M, Q, dt in [("c1", 1024, 64, "fp32"), ("c3", 3001, 150, "bf16"), ("c2", 700, 37, "bf16"),
                       ("c4", 513, 260, "bf16")]:
    cfg = ams_gen.CONFIGS["c1"] if name == "c1" else ams_gen.small_variant(name, M, Q)
    w = ams_gen.generate_host(cfg)
    with ams.Pool(w.emb.shape[1], cfg.J, cfg.M, cfg.Q, 64, dtype=dt, shard_block=256) as pool:
        pool.append(T(w.emb), T(w.joints))
        for gamma in (cfg.gamma, INF):
            for k in (cfg.k, 33):
                for gf in ((False, True) if dt == "bf16" else (False,)):
                    out = pool.match(T(w.q_emb), T(w.q_joints), k, cfg.theta, gamma, gate_first=gf)
                    torch.cuda.synchronize()
                    orc = oracle.match(w.emb, w.joints, w.q_emb, w.q_joints, k, cfg.theta, gamma)
                    g = [t.cpu().numpy() for t in out]
                    (check_exact(*g, orc) if dt == "fp32" else check_bf16(*g, orc, cfg.theta))
# small-batch kernel: one CTA (nq <= 128), CTA pairs narrow and wide (129-256 queries, k <= 8),
# ungated and gated; auto route
cfg = ams_gen.small_variant("c3", 1300, 200)
w = ams_gen.generate_host(cfg)
with ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, 8) as pool:
    pool.append(T(w.emb), T(w.joints))
    for nq, pol in ((60, 0), (200, 8), (200, 12)):
        ams.ams_pool_set_kernel_policy(pool.handle, pol)
        for gamma in (0.3, 3.5, INF):
            out = pool.match(T(w.q_emb[:nq]), T(w.q_joints[:nq]), 8, cfg.theta, gamma)
            torch.cuda.synchronize()
            assert ams.ams_pool_last_plan(pool.handle)["kernel_id"] == 4
            orc = oracle.match(w.emb, w.joints, w.q_emb[:nq], w.q_joints[:nq], 8, cfg.theta, gamma)
            check_bf16(*[t.cpu().numpy() for t in out], orc, cfg.theta)
    ams.ams_pool_set_kernel_policy(pool.handle, 0)
    out = pool.match(T(w.q_emb), T(w.q_joints), 8, cfg.theta, 0.3, gate_first="auto")
    torch.cuda.synchronize()
# peer-exchange kernels (virtual ranks, late-consumer order)
G, nq, k, rounds = 3, 33, 8, 3
sx = torch.sort(torch.rand(rounds, G, nq, k, device="cuda"), dim=3, descending=True).values.contiguous()
ix = torch.arange(rounds * G * nq * k, device="cuda", dtype=torch.int64).reshape(rounds, G, nq, k).contiguous()
ox = torch.empty(rounds, G, nq, k, device="cuda"); oix = torch.empty(rounds, G, nq, k, dtype=torch.int64, device="cuda")
ohx = torch.empty(rounds, G, nq, dtype=torch.uint8, device="cuda")
ams.ams_exchange_selftest(G, nq, k, rounds, 0.5, sx, ix, ox, oix, ohx, flags=ams.AMS_SELFTEST_LATE_CONSUMER)
# merge entry
s = torch.sort(torch.rand(3, 50, 8, device="cuda"), dim=2, descending=True).values.contiguous()
i = torch.arange(3 * 50 * 8, device="cuda", dtype=torch.int64).reshape(3, 50, 8).contiguous()
oi = torch.empty(50, 8, dtype=torch.int64, device="cuda"); os_ = torch.empty(50, 8, device="cuda")
oh = torch.empty(50, dtype=torch.uint8, device="cuda")
ams.ams_merge_topk(s, i, 3, 50, 8, 8, 0.5, oi, os_, oh)
# hash + store
rng = np.random.Generator(np.random.PCG64(3))
lens = rng.integers(0, 9000, 30); offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64) + 5
data = rng.integers(0, 256, int(offs[-1]) + 1, dtype=np.uint8)
h = ams.ams_hasher_create(0, 30, int(offs[-1]), 4096)
out = torch.empty(30, dtype=torch.int64, device="cuda")
ams.ams_hash_actions(h, T(data), offs, 30, out); torch.cuda.synchronize()
assert np.array_equal(out.cpu().numpy().view(np.uint64), oracle.hash_actions(data, offs))
ams.ams_hasher_destroy(h)
# tensor-core hash path: 16-B aligned inputs with full 4 KB segments
lens = (rng.integers(0, 3 * 4096, 40) // 16) * 16
offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
data = rng.integers(0, 256, int(offs[-1]) + 16, dtype=np.uint8)
h = ams.ams_hasher_create(0, 40, int(offs[-1]), 4096)
out = torch.empty(40, dtype=torch.int64, device="cuda")
ams.ams_hash_actions(h, T(data), offs, 40, out); torch.cuda.synchronize()
assert ams.ams_hasher_last_stats(h)["tc_segments"] > 0
assert np.array_equal(out.cpu().numpy().view(np.uint64), oracle.hash_actions(data, offs))
ams.ams_hasher_destroy(h)
st = ams.ams_vstore_create(0, 256, 1 << 20, 64, 1 << 20)
acts = [bytes(rng.integers(0, 256, rng.integers(0, 500), dtype=np.uint8)) for _ in range(20)]
batch = [acts[j] for j in rng.integers(0, 20, 64)]
o2 = np.concatenate([[0], np.cumsum([len(a) for a in batch])]).astype(np.int64)
d2 = np.frombuffer(b"".join(batch), np.uint8).copy()
ids = torch.empty(64, dtype=torch.int64, device="cuda"); stt = torch.empty(64, dtype=torch.uint8, device="cuda")
ams.ams_vstore_intern(st, d2, o2, 64, None, ids, stt)
rem = torch.empty(64, dtype=torch.int64, device="cuda")
ams.ams_vstore_release(st, ids, 64, rem)
ams.ams_vstore_compact(st)
ams.ams_vstore_stats(st); ams.ams_vstore_destroy(st)
torch.cuda.synchronize()
print("memcheck cases: ok")
