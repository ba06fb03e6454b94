"""Object lifecycles release their device memory: pools (dense, small-batch, gate-first with
its lazily built joint-0 snapshot and query bins, the auto route's estimate), hashers and
virtual-action stores are created, used and destroyed 12 times, and the device's free
memory returns to where it started (within the slack of the CUDA context's own
bookkeeping).  A leak of one pool's buffers per cycle would be hundreds of MB."""
import numpy as np
import pytest

import ams_gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def free_bytes():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return torch.cuda.mem_get_info()[0]


def one_cycle(ams, w, cfg):
    dev = torch.device("cuda", 0)
    with ams.Pool(cfg.d, cfg.J, cfg.M, cfg.Q, cfg.k, dtype="bf16") as pool:
        pool.append(T(w.emb), T(w.joints))
        q, qj = T(w.q_emb).view(torch.bfloat16), T(w.q_joints)
        for nq, route in ((cfg.Q, False), (64, False), (1, True), (40, True), (cfg.Q, True), (64, "auto")):
            out = pool.match(q[:nq].contiguous(), qj[:nq].contiguous(), cfg.k, cfg.theta, cfg.gamma, gate_first=route)
            del out
    h = ams.ams_hasher_create(0, 8, 1 << 16, 4096)
    data = torch.randint(0, 256, (1 << 16,), dtype=torch.uint8, device=dev)
    offs = np.array([0, 4096, 9000, 1 << 16], np.int64)
    hout = torch.empty(3, dtype=torch.int64, device=dev)
    ams.ams_hash_actions(h, data, offs, 3, hout)
    ams.ams_hasher_destroy(h)
    st = ams.ams_vstore_create(0, 256, 1 << 20, 64, 1 << 16)
    ams.ams_vstore_destroy(st)
    torch.cuda.synchronize()


def test_create_use_destroy_returns_device_memory(ams):
    # a pool above the 64 K-row snapshot threshold, so the gate-first calls build the index
    cfg = ams_gen.small_variant("c2", 70000, 200)
    w = ams_gen.generate_host(cfg)
    one_cycle(ams, w, cfg)             # first use: CUDA module loading, cuBLAS-free lazy state
    base = free_bytes()
    for _ in range(12):
        one_cycle(ams, w, cfg)
    drift = base - free_bytes()
    assert drift < 64 << 20, f"{drift / 2**20:.1f} MiB of device memory not returned after 12 cycles"
