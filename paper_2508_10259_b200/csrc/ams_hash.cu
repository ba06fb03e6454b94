// ams_hash.cu -- GPU two-phase hashing for the action index.
//
// PAPER.md:538-543 (3.2.3) and Algorithm 1 `lst:impl:index`:
//   Phase 1: "independently calculates a hash value for each segment using parallelism"
//   Phase 2: "merges all the segments' hash values to generate the final hash result"
//   "the hash functions involved are modular calculation"
// Concretised by SPEC.md:103-111 (and used bit-exactly here): B = 257, M = 2^61 - 1,
// segment size s (default 4096 B); h_i = polynomial hash of segment i's bytes
// (h = h*B + byte mod M from 0); H_final = fold (acc*B + h_i) mod M from 0; empty -> 0.
//
// GPU mapping.  Phase 1: one warp per segment.  The segment splits into an unaligned
// head (< 16 B), 16-byte pieces and a tail (< 16 B): value = ((H_head * B^(16P) + H_body)
// * B^tail + H_tail).  Lane l loads pieces l, l+32, ... with coalesced 16-B loads; a
// piece hashes as four 4-byte groups G = ((b0*B + b1)*B + b2)*B + b3 folded by B^4; the
// lane keeps a Horner sum in steps of B^512 and scales it by B^(16*(P-1-last piece));
// a butterfly sums the lanes mod M.  Phase 2: one warp per input folds its k segment
// hashes the same way (steps of B^32).  All arithmetic is exact modular arithmetic on
// 64-bit limbs (Mersenne reduction), so the result is bit-identical to the sequential
// definition for every input.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/ams.h"

namespace ams {
namespace hash {

constexpr uint64_t kM = (uint64_t(1) << 61) - 1;
constexpr uint64_t kB = 257;

__host__ __device__ __forceinline__ uint64_t red(uint64_t x) { return (x & kM) + (x >> 61); }
__host__ __device__ __forceinline__ uint64_t canon(uint64_t x) {
  x = red(red(x));
  return x >= kM ? x - kM : x;
}
// a < 2^62, c < 2^61: a*c mod M, result < 2^61 + 8 (lazy)
__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t c) {
  const uint64_t lo = a * c;
  const uint64_t hi = __umul64hi(a, c);
  return red((lo & kM) + (lo >> 61) + (hi << 3));
}
__host__ uint64_t mulmod_host(uint64_t a, uint64_t c) {
  const unsigned __int128 p = (unsigned __int128)a * c;
  return (uint64_t)(p % kM);
}
__device__ __forceinline__ uint64_t powmod(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r = mulmod(r, b);
    b = mulmod(b, b);
    e >>= 1;
  }
  return r;
}
// Horner over n (< 16) bytes starting from h
__device__ __forceinline__ uint64_t horner_bytes(uint64_t h, const uint8_t* p, int n) {
  for (int i = 0; i < n; ++i) h = red(mulmod(h, kB) + p[i]);
  return h;
}
// G(word) for the 4 bytes of a little-endian 32-bit word, in address order
__device__ __forceinline__ uint64_t g4(uint32_t w) {
  const uint32_t b0 = w & 0xFF, b1 = (w >> 8) & 0xFF, b2 = (w >> 16) & 0xFF, b3 = w >> 24;
  return (uint64_t)((b0 * 257u + b1) * 257u + b2) * 257u + b3;   // < 2^33
}
__device__ __forceinline__ uint64_t warp_sum_mod(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = red(v + __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fast path weights (full, 16-B aligned segments of 512*J bytes, J <= 8): the lane's
// value is sum_j sum_u G2(j,u) * E[J-1-j][u] with G2 = b0*B + b1 the 2-byte groups of its
// j-th 16-byte piece and E[jj][u] = B^(2(7-u)) * B^(512 jj) mod M (= the Horner weights
// of the slow path, expanded).  Split into 32-bit halves so every product is a single
// 32x32->64 multiply-add with no reduction until the end.
__constant__ uint32_t kE_lo[8][8];
__constant__ uint32_t kE_hi[8][8];

struct Tables {
  const uint64_t* pow16;   // B^(16 e) mod M, e = 0..s/16
  uint64_t B4, B512, B32;
  uint64_t pow1[16];       // B^t, t < 16
};

__global__ void phase1_kernel(const uint8_t* __restrict__ data, const int64_t* __restrict__ offsets,
                              const int64_t* __restrict__ seg_base, int32_t n_inputs, int64_t n_segs, int64_t s,
                              Tables tb, uint64_t* __restrict__ seg_hash) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  // each warp takes a contiguous run of segments: one binary search for the owning
  // input of its first segment, then a forward walk (no dependent search per segment)
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t per = (n_segs + warps - 1) / warps;
  const int64_t g_begin = wid * per, g_end = min(n_segs, g_begin + per);
  int lo = 0;
  if (g_begin < g_end) {   // input owning segment g_begin: last i with seg_base[i] <= g
    int hi = n_inputs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (seg_base[mid] <= g_begin) lo = mid; else hi = mid - 1;
    }
  }
  int64_t next_base = g_begin < g_end ? seg_base[lo + 1] : 0;
  for (int64_t g = g_begin; g < g_end; ++g) {
    while (g >= next_base) next_base = seg_base[++lo + 1];   // skips empty inputs
    const int64_t j = g - seg_base[lo];
    const int64_t start = offsets[lo] + j * s;
    const int64_t len = min(s, offsets[lo + 1] - start);
    const uint8_t* p = data + start;
    const int head = (int)min(len, (int64_t)((16 - ((uintptr_t)p & 15)) & 15));
    const int64_t P = (len - head) >> 4;
    const int tail = (int)(len - head - 16 * P);
    const uint4* body = reinterpret_cast<const uint4*>(p + head);
    uint64_t acc = 0;
    int64_t last = -1;
    if (head == 0 && tail == 0 && (P & 31) == 0 && P > 0 && P <= 256) {
      // lazy accumulation: sum < 64 * 2^49 (lo) and 64 * 2^46 (hi), reduced once
      const int J = (int)(P >> 5);
      uint64_t lo = 0, hi = 0;
      auto piece = [&](const uint4 w, int jj) {
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) {
          const uint32_t ga = (ws[wi] & 0xFFu) * 257u + ((ws[wi] >> 8) & 0xFFu);
          const uint32_t gb = ((ws[wi] >> 16) & 0xFFu) * 257u + (ws[wi] >> 24);
          lo += (uint64_t)ga * kE_lo[jj][2 * wi] + (uint64_t)gb * kE_lo[jj][2 * wi + 1];
          hi += (uint64_t)ga * kE_hi[jj][2 * wi] + (uint64_t)gb * kE_hi[jj][2 * wi + 1];
        }
      };
      if (J == 8) {   // the default 4 KB segment: all eight 16-B loads in flight at once
        uint4 w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = __ldg(body + lane + 32 * j);
#pragma unroll
        for (int j = 0; j < 8; ++j) piece(w[j], 7 - j);
      } else {
        for (int j = 0; j < J; ++j) piece(__ldg(body + lane + 32 * j), J - 1 - j);
      }
      // hi * 2^32 = (hi >> 29) * 2^61 + (hi mod 2^29) * 2^32, and 2^61 = 1 (mod M)
      acc = red(red(lo) + (hi >> 29) + ((hi & 0x1FFFFFFFull) << 32));
      last = lane + 32 * (J - 1);
    } else
    for (int64_t q = lane; q < P; q += 32) {
      const uint4 w = __ldg(body + q);
      uint64_t h = g4(w.x);
      h = red(mulmod(h, tb.B4) + g4(w.y));
      h = red(mulmod(h, tb.B4) + g4(w.z));
      h = red(mulmod(h, tb.B4) + g4(w.w));
      acc = red(mulmod(acc, tb.B512) + h);
      last = q;
    }
    if (last >= 0) acc = mulmod(acc, tb.pow16[P - 1 - last]);
    acc = warp_sum_mod(acc);
    if (lane == 0) {
      uint64_t v = horner_bytes(0, p, head);
      v = red(mulmod(v, tb.pow16[P]) + acc);
      v = horner_bytes(v, p + head + 16 * P, tail);
      seg_hash[g] = canon(v);
    }
  }
}

__global__ void phase2_kernel(const int64_t* __restrict__ seg_base, int32_t n_inputs,
                              const uint64_t* __restrict__ seg_hash, Tables tb, uint64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n_inputs) return;
  const int64_t b0 = seg_base[i], k = seg_base[i + 1] - b0;
  uint64_t acc = 0;
  int64_t last = -1;
  for (int64_t j = lane; j < k; j += 32) {
    acc = red(mulmod(acc, tb.B32) + seg_hash[b0 + j]);
    last = j;
  }
  if (last >= 0) acc = mulmod(acc, powmod(kB, (uint64_t)(k - 1 - last)));
  acc = warp_sum_mod(acc);
  if (lane == 0) out[i] = canon(acc);
}

}  // namespace hash
}  // namespace ams

struct ams_hasher_s {
  int32_t device = 0;
  int64_t max_inputs = 0, max_bytes = 0, s = 4096, max_segs = 0;
  uint8_t* d_stage = nullptr;
  int64_t* d_offsets = nullptr;
  int64_t* d_seg_base = nullptr;
  uint64_t* d_seg_hash = nullptr;
  uint64_t* d_pow16 = nullptr;
  int64_t* h_pinned = nullptr;   // [2 * (max_inputs + 1)]: offsets, seg_base
  cudaEvent_t done = nullptr;
  bool pending = false;
  bool broken = false;
  ams::hash::Tables tb{};
};

namespace {
void hasher_free(ams_hasher_s* h) {
  if (!h) return;
  cudaFree(h->d_stage);
  cudaFree(h->d_offsets);
  cudaFree(h->d_seg_base);
  cudaFree(h->d_seg_hash);
  cudaFree(h->d_pow16);
  if (h->h_pinned) cudaFreeHost(h->h_pinned);
  if (h->done) cudaEventDestroy(h->done);
  delete h;
}
bool dev_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
}  // namespace

extern "C" {

ams_status_t ams_hasher_create(int32_t device, int64_t max_inputs, int64_t max_bytes, int64_t segment_size,
                               ams_hasher_t* out) {
  using namespace ams::hash;
  if (out == nullptr || max_inputs < 1 || max_bytes < 0 || segment_size < 1 || segment_size > (1 << 24))
    return AMS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return AMS_ERR_INVALID_ARGUMENT;
  }
  if (cudaSetDevice(device) != cudaSuccess) return AMS_ERR_CUDA;
  auto* h = new (std::nothrow) ams_hasher_s;
  if (!h) return AMS_ERR_OUT_OF_MEMORY;
  h->device = device;
  h->max_inputs = max_inputs;
  h->max_bytes = max_bytes;
  h->s = segment_size;
  h->max_segs = max_bytes / segment_size + max_inputs + 1;
  const int64_t npow = segment_size / 16 + 2;
  bool ok = cudaMalloc(&h->d_stage, std::max<int64_t>(max_bytes, 16)) == cudaSuccess &&
            cudaMalloc(&h->d_offsets, (max_inputs + 1) * sizeof(int64_t)) == cudaSuccess &&
            cudaMalloc(&h->d_seg_base, (max_inputs + 1) * sizeof(int64_t)) == cudaSuccess &&
            cudaMalloc(&h->d_seg_hash, h->max_segs * sizeof(uint64_t)) == cudaSuccess &&
            cudaMalloc(&h->d_pow16, npow * sizeof(uint64_t)) == cudaSuccess &&
            cudaMallocHost(&h->h_pinned, 2 * (max_inputs + 1) * sizeof(int64_t)) == cudaSuccess &&
            cudaEventCreateWithFlags(&h->done, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    hasher_free(h);
    return AMS_ERR_OUT_OF_MEMORY;
  }
  // power tables (host, exact 128-bit arithmetic)
  std::vector<uint64_t> pw(npow);
  uint64_t b16 = 1;
  for (int i = 0; i < 16; ++i) b16 = mulmod_host(b16, kB);
  pw[0] = 1;
  for (int64_t e = 1; e < npow; ++e) pw[e] = mulmod_host(pw[e - 1], b16);
  h->tb.pow1[0] = 1;
  for (int t = 1; t < 16; ++t) h->tb.pow1[t] = mulmod_host(h->tb.pow1[t - 1], kB);
  h->tb.B4 = mulmod_host(mulmod_host(kB, kB), mulmod_host(kB, kB));
  uint64_t b512 = 1, b32 = 1;
  for (int i = 0; i < 512; ++i) b512 = mulmod_host(b512, kB);
  for (int i = 0; i < 32; ++i) b32 = mulmod_host(b32, kB);
  h->tb.B512 = b512;
  h->tb.B32 = b32;
  if (cudaMemcpy(h->d_pow16, pw.data(), npow * sizeof(uint64_t), cudaMemcpyHostToDevice) != cudaSuccess) {
    hasher_free(h);
    return AMS_ERR_CUDA;
  }
  h->tb.pow16 = h->d_pow16;
  {  // fast-path weights E[jj][u] = B^(2(7-u)) * B^(512 jj) mod M
    uint32_t elo[8][8], ehi[8][8];
    uint64_t bj = 1;   // B^(512 jj)
    for (int jj = 0; jj < 8; ++jj) {
      for (int u = 0; u < 8; ++u) {
        uint64_t w = bj;
        for (int e = 0; e < 2 * (7 - u); ++e) w = mulmod_host(w, kB);
        elo[jj][u] = (uint32_t)(w & 0xFFFFFFFFull);
        ehi[jj][u] = (uint32_t)(w >> 32);
      }
      bj = mulmod_host(bj, b512);
    }
    if (cudaMemcpyToSymbol(kE_lo, elo, sizeof elo) != cudaSuccess ||
        cudaMemcpyToSymbol(kE_hi, ehi, sizeof ehi) != cudaSuccess) {
      hasher_free(h);
      return AMS_ERR_CUDA;
    }
  }
  *out = h;
  return AMS_OK;
}

ams_status_t ams_hash_actions(ams_hasher_t h, const uint8_t* data, const int64_t* offsets, int32_t n_inputs,
                              uint64_t* out_hash, void* stream) {
  if (h == nullptr || offsets == nullptr || out_hash == nullptr || n_inputs < 1 || n_inputs > h->max_inputs)
    return AMS_ERR_INVALID_ARGUMENT;
  if (h->broken) return AMS_ERR_CUDA;
  const int64_t total = offsets[n_inputs] - offsets[0];
  if (offsets[0] < 0 || total < 0 || (total > 0 && data == nullptr)) return AMS_ERR_INVALID_ARGUMENT;
  const bool device_data = total > 0 && dev_ptr(data);
  if (total > h->max_bytes) return AMS_ERR_CAPACITY;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaSetDevice(h->device) != cudaSuccess) return AMS_ERR_CUDA;
  // the pinned staging buffer is reused: wait until the previous call consumed it
  if (h->pending && cudaEventSynchronize(h->done) != cudaSuccess) {
    h->broken = true;
    return AMS_ERR_CUDA;
  }
  int64_t* off = h->h_pinned;
  int64_t* base = h->h_pinned + (h->max_inputs + 1);
  int64_t nseg = 0;
  for (int32_t i = 0; i <= n_inputs; ++i) {
    off[i] = device_data ? offsets[i] : offsets[i] - offsets[0];
    if (i > 0 && offsets[i] < offsets[i - 1]) return AMS_ERR_INVALID_ARGUMENT;
  }
  for (int32_t i = 0; i < n_inputs; ++i) {
    base[i] = nseg;
    nseg += (offsets[i + 1] - offsets[i] + h->s - 1) / h->s;
  }
  base[n_inputs] = nseg;
  if (nseg > h->max_segs) return AMS_ERR_CAPACITY;
  const uint8_t* src = data;
  bool ok = cudaMemcpyAsync(h->d_offsets, off, (n_inputs + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s) ==
                cudaSuccess &&
            cudaMemcpyAsync(h->d_seg_base, base, (n_inputs + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s) ==
                cudaSuccess;
  if (ok && total > 0 && !device_data) {
    ok = cudaMemcpyAsync(h->d_stage, data + offsets[0], total, cudaMemcpyDefault, s) == cudaSuccess;
    src = h->d_stage;
  }
  if (ok && nseg > 0) {
    const int wpb = 8;
    const int64_t blocks = std::min<int64_t>((nseg + wpb - 1) / wpb, 148 * 16);
    ams::hash::phase1_kernel<<<(unsigned)blocks, wpb * 32, 0, s>>>(src, h->d_offsets, h->d_seg_base, n_inputs, nseg,
                                                                   h->s, h->tb, h->d_seg_hash);
    ok = cudaGetLastError() == cudaSuccess;
  }
  if (ok) {
    const int wpb = 8;
    ams::hash::phase2_kernel<<<(unsigned)((n_inputs + wpb - 1) / wpb), wpb * 32, 0, s>>>(
        h->d_seg_base, n_inputs, h->d_seg_hash, h->tb, out_hash);
    ok = cudaGetLastError() == cudaSuccess;
  }
  ok = ok && cudaEventRecord(h->done, s) == cudaSuccess;
  if (!ok) {
    h->broken = true;
    return AMS_ERR_CUDA;
  }
  h->pending = true;
  return AMS_OK;
}

ams_status_t ams_hasher_destroy(ams_hasher_t h) {
  if (h == nullptr) return AMS_OK;
  cudaSetDevice(h->device);
  const ams_status_t st = cudaDeviceSynchronize() == cudaSuccess ? AMS_OK : AMS_ERR_CUDA;
  hasher_free(h);
  return st;
}

}  // extern "C"
