"""GPU two-phase action hash vs the oracle, bit for bit."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ams():
    import paper_2508_10259_b200 as m
    return m


def _csr(rng, lens, pad=0):
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    data = rng.integers(0, 256, int(offs[-1]) + 1 + pad, dtype=np.uint8)
    return data, offs


def _gpu_hash(ams, data, offs, s, device_data):
    n = len(offs) - 1
    h = ams.ams_hasher_create(0, n, max(int(offs[-1]), 1), s)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    src = torch.from_numpy(data).cuda() if device_data else data
    ams.ams_hash_actions(h, src, offs, n, out)
    torch.cuda.synchronize()
    ams.ams_hasher_destroy(h)
    return out.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("s", [4096, 64, 16, 1, 10000])
@pytest.mark.parametrize("device_data", [False, True])
def test_hash_random_batches(ams, s, device_data):
    rng = np.random.Generator(np.random.PCG64(s))
    lens = np.concatenate([[0, 1, 15, 16, 17, 31, 4095, 4096, 4097, 8192, 100_003, 0],
                           rng.integers(0, 20000, 60)])
    data, offs = _csr(rng, lens, pad=3)
    offs = offs + 3            # every input starts unaligned (data is 3 bytes longer)
    exp = oracle.hash_actions(data, offs, s=s)
    got = _gpu_hash(ams, data, offs, s, device_data)
    assert np.array_equal(got, exp)


def test_hash_large_blob_and_many_small(ams):
    rng = np.random.Generator(np.random.PCG64(1))
    blob = 64 << 20    # a 64 MB blob (KV-cache sized, Table 1) + 20k 57-byte actions
    lens = np.concatenate([[blob], np.full(20000, 57)])
    data, offs = _csr(rng, lens)
    exp = oracle.hash_actions(data, offs)
    got = _gpu_hash(ams, data, offs, 4096, True)
    assert np.array_equal(got, exp)
    assert len(set(got[1:].tolist())) == 20000          # distinct random actions -> distinct ids


def test_hash_all_ff_and_zero(ams):
    data = np.concatenate([np.full(300000, 255, np.uint8), np.zeros(300000, np.uint8)])
    offs = np.array([0, 300000, 600000, 600000], np.int64)
    exp = oracle.hash_actions(data, offs)
    got = _gpu_hash(ams, data, offs, 4096, False)
    assert np.array_equal(got, exp) and got[1] == 0 and got[2] == 0


def test_hash_errors(ams):
    h = ams.ams_hasher_create(0, 4, 100, 4096)
    out = torch.empty(4, dtype=torch.int64, device="cuda")
    data = np.zeros(200, np.uint8)
    with pytest.raises(ams.AmsError) as e:
        ams.ams_hash_actions(h, data, np.array([0, 150], np.int64), 1, out)   # host bytes > max_bytes
    assert e.value.status == 2
    with pytest.raises(ams.AmsError) as e:
        ams.ams_hash_actions(h, data, np.array([0, 10, 5], np.int64), 2, out)  # decreasing offsets
    assert e.value.status == 1
    with pytest.raises(ams.AmsError) as e:
        ams.ams_hash_actions(h, data, np.zeros(6, np.int64), 5, out)            # n_inputs > max_inputs
    assert e.value.status == 1
    ams.ams_hasher_destroy(h)


def _gpu_hash_stats(ams, data, offs, s, device_data):
    n = len(offs) - 1
    h = ams.ams_hasher_create(0, n, max(int(offs[-1]), 1), s)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    src = torch.from_numpy(data).cuda() if device_data else data
    ams.ams_hash_actions(h, src, offs, n, out)
    torch.cuda.synchronize()
    st = ams.ams_hasher_last_stats(h)
    ams.ams_hasher_destroy(h)
    return out.cpu().numpy().view(np.uint64), st


@pytest.mark.parametrize("s", [128, 4096, 8192])
@pytest.mark.parametrize("fill", ["random", "ff"])
def test_hash_tensor_core_path_exact(ams, s, fill):
    """Full 16-B aligned segments take the tcgen05 kind::i8 path (u8 bytes x 8-bit limbs of
    B^(s-1-k) mod M, s32 accumulate, fold mod M); bit-exact against the sequential oracle,
    including all-0xFF bytes (the largest limb sums) and inputs with partial last segments."""
    rng = np.random.Generator(np.random.PCG64(s + (fill == "ff")))
    lens = np.array([16 * int(x) for x in rng.integers(0, 6 * s // 16, 40)] + [s, 2 * s, 3 * s + 16, 0, 16], np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)   # every input 16-B aligned
    data = (np.full(int(offs[-1]) + 16, 255, np.uint8) if fill == "ff"
            else rng.integers(0, 256, int(offs[-1]) + 16, dtype=np.uint8))
    exp = oracle.hash_actions(data, offs, s=s)
    for device_data in (False, True):
        got, st = _gpu_hash_stats(ams, data, offs, s, device_data)
        assert np.array_equal(got, exp), device_data
        assert st["tc_segments"] == int(np.sum(lens // s)) > 0
        assert st["segments"] == int(np.sum((lens + s - 1) // s))


def test_hash_tensor_core_mixed_alignment(ams):
    """Aligned and unaligned inputs in one batch: each segment is hashed by exactly one of
    the two phase-1 kernels (tensor-core for full aligned segments, CUDA cores otherwise)."""
    rng = np.random.Generator(np.random.PCG64(9))
    lens = rng.integers(0, 5 * 4096, 200)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    data = rng.integers(0, 256, int(offs[-1]) + 1, dtype=np.uint8)
    exp = oracle.hash_actions(data, offs)
    got, st = _gpu_hash_stats(ams, data, offs, 4096, True)
    assert np.array_equal(got, exp)
    aligned = (offs[:-1] % 16) == 0
    assert st["tc_segments"] == int(np.sum((lens // 4096)[aligned])) > 0
    assert st["tc_segments"] < st["segments"]


def test_hash_tensor_core_many_tiles(ams):
    """More 128-segment tiles than SMs (the persistent loop wraps, TMEM double buffer and
    every shared-memory stage reused many times): 48 x 4 MB aligned inputs."""
    rng = np.random.Generator(np.random.PCG64(3))
    lens = np.full(48, 4 << 20, np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    data = rng.integers(0, 256, int(offs[-1]), dtype=np.uint8)
    exp = oracle.hash_actions(data, offs)
    got, st = _gpu_hash_stats(ams, data, offs, 4096, True)
    assert np.array_equal(got, exp)
    assert st["tc_segments"] == st["segments"] == 48 * 1024
