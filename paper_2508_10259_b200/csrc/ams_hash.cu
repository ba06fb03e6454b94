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
//
// Tensor-core phase 1 (full, 16-B aligned segments; s a multiple of 128, s <= 8192).  A
// segment's hash is a dot product: h = sum_k b_k w_k mod M with w_k = B^(s-1-k) mod M
// (Horner expanded).  Split every w_k into eight 8-bit limbs w_k = sum_n w_kn 2^(8n):
// h = sum_n 2^(8n) S_n mod M, S_n = sum_k b_k w_kn -- an exact u8 x u8 -> s32 contraction
// (S_n <= 8192 * 255 * 255 < 2^31) of the [segments x s] byte matrix with the constant
// [s x 8] limb matrix: tcgen05.mma kind::i8, M = 128 segments, N = 8 limbs, K = 32 per
// instruction, accumulators in TMEM.  The segment bytes are streamed from HBM once; the
// limb matrix stays in shared memory; the epilogue folds the 8 limb sums mod M.  Segments
// start at arbitrary 16-B aligned offsets (CSR inputs), so they are staged with 16-byte
// cp.async into the 128-B-swizzled K-major layout rather than by a tensor map.  Every
// other segment (partial, unaligned) keeps the CUDA-core path above; both write the
// same per-segment hash array, so phase 2 is unchanged.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/ams.h"
#include "ams_ptx.cuh"

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

// Segments the tensor-core kernel hashes (identical test in both phase-1 kernels).
__device__ __forceinline__ bool tc_segment(const uint8_t* data, int64_t start, int64_t len, int64_t s, int tc_on) {
  return tc_on != 0 && len == s && ((reinterpret_cast<uintptr_t>(data + start) & 15u) == 0);
}

// owning input of segment g: last i with seg_base[i] <= g (empty inputs share a base)
__device__ __forceinline__ int owner_of(const int64_t* __restrict__ seg_base, int32_t n_inputs, int64_t g) {
  int lo = 0, hi = n_inputs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg_base[mid] <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}

constexpr int kTcRows = 128;                     // segments per tile (MMA M)
constexpr int kTcLimbs = 8;                      // MMA N
constexpr int kTcStages = 8;                     // 16 KB A stages
constexpr int kTcLag = 6;                        // cp.async groups in flight per producer thread
constexpr int kTcProducerWarps = 4;
constexpr int kTcEpiWarps = 4;
constexpr int kTcThreads = 32 * (kTcProducerWarps + 1 + kTcEpiWarps);   // 288
constexpr uint32_t kTcStageBytes = kTcRows * 128;                       // 16 KB
constexpr int kTcMaxKb = 64;                                            // s <= 8192
__host__ __device__ constexpr uint32_t tc_smem_bytes(int n_kb) {
  return 1024 + (uint32_t)n_kb * 1024 + kTcStages * kTcStageBytes + 256;
}

// wgt: [n_kb][8 limbs][128 B] in the 128-B swizzled K-major layout (host-built)
__global__ void __launch_bounds__(kTcThreads, 1)
    phase1_tc_kernel(const uint8_t* __restrict__ data, const int64_t* __restrict__ offsets,
                     const int64_t* __restrict__ seg_base, int32_t n_inputs, int64_t n_segs, int64_t s,
                     const uint8_t* __restrict__ wgt, uint64_t* __restrict__ seg_hash) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int n_kb = (int)(s / 128);
  uint8_t* sB = smem;                                   // n_kb KB
  uint8_t* sA = smem + n_kb * 1024;                     // kTcStages x 16 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + kTcStages * kTcStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kTcStages;
  uint64_t* tfull = bars + 2 * kTcStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kMmaWarp = kTcProducerWarps;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kTcStages; ++i) {
      ptx::mbar_init(&full[i], 32 * kTcProducerWarps);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kTcEpiWarps);
    }
    ptx::fence_mbar_init();
  }
  // the constant limb matrix -> shared memory (already in the swizzled layout)
  for (int i = threadIdx.x; i < n_kb * 64; i += kTcThreads)
    reinterpret_cast<uint4*>(sB)[i] = __ldg(reinterpret_cast<const uint4*>(wgt) + i);
  ptx::fence_proxy_async_smem();
  if (warp == kMmaWarp) {
    ptx::tmem_alloc<1>(tmem_holder, 32);
    ptx::tmem_relinquish<1>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int64_t n_tiles = (n_segs + kTcRows - 1) / kTcRows;

  if (warp < kTcProducerWarps) {
    // ------------------------------------------------------------ cp.async producers
    // warp pw stages rows 32 pw .. 32 pw + 31; instruction i covers rows 32 pw + 4 i +
    // lane / 8, 16-byte chunk lane % 8 of the K-block (4 full 128-B rows per instruction)
    const int pw = warp;
    const int chunk = lane & 7;
    uint32_t dst_off[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 32 * pw + 4 * i + (lane >> 3);
      dst_off[i] = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((chunk ^ (r & 7)) << 4));
    }
    const uint32_t sA_u = ptx::smem_u32(sA);
    uint32_t it = 0;   // stage sequence number
    for (int64_t T = blockIdx.x; T < n_tiles; T += gridDim.x) {
      const int64_t g = T * kTcRows + 32 * pw + lane;
      const uint8_t* rp = nullptr;
      int el = 0;
      if (g < n_segs) {
        const int i = owner_of(seg_base, n_inputs, g);
        const int64_t start = offsets[i] + (g - seg_base[i]) * s;
        const int64_t len = min(s, offsets[i + 1] - start);
        el = tc_segment(data, start, len, s, 1) ? 1 : 0;
        rp = data + start;
      }
      const uint8_t* src[8];
      int ok = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int sl = 4 * i + (lane >> 3);
        src[i] = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(rp), sl)) +
                 16 * chunk;
        ok |= __shfl_sync(0xffffffffu, el, sl) << i;
      }
      for (int kb = 0; kb < n_kb; ++kb, ++it) {
        const uint32_t slot = it % kTcStages;
        ptx::mbar_wait(&empty[slot], ((it / kTcStages) & 1u) ^ 1u);
        const uint32_t base = sA_u + slot * kTcStageBytes;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if ((ok >> i) & 1) ptx::cp_async16(base + dst_off[i], src[i] + 128 * kb);
        ptx::cp_async_commit();
        if (it >= kTcLag) {   // stage it - kTcLag has landed: publish it to the MMA
          ptx::cp_async_wait<kTcLag>();
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive(&full[(it - kTcLag) % kTcStages]);
        }
      }
    }
    ptx::cp_async_wait<0>();
    ptx::fence_proxy_async_smem();
    for (uint32_t j = it > (uint32_t)kTcLag ? it - kTcLag : 0; j < it; ++j) ptx::mbar_arrive(&full[j % kTcStages]);
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = ptx::idesc_u8_s32(kTcRows, kTcLimbs);
    const uint64_t da0 = ptx::sdesc_k_sw128(ptx::smem_u32(sA));
    const uint64_t db0 = ptx::sdesc_k_sw128(ptx::smem_u32(sB));
    uint32_t it = 0, tcount = 0;
    for (int64_t T = blockIdx.x; T < n_tiles; T += gridDim.x, ++tcount) {
      const uint32_t buf = tcount & 1u;
      ptx::mbar_wait(&tempty[buf], ((tcount >> 1) & 1u) ^ 1u);
      ptx::tc_fence_after();
      const uint32_t d = tmem_base + buf * kTcLimbs;
      for (int kb = 0; kb < n_kb; ++kb, ++it) {
        const uint32_t slot = it % kTcStages;
        ptx::mbar_wait(&full[slot], (it / kTcStages) & 1u);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint64_t da = da0 + (uint64_t)(slot * (kTcStageBytes >> 4));
          const uint64_t db = db0 + (uint64_t)(kb * (1024 >> 4));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)   // K = 32 bytes per instruction: +32 B = +2 in the descriptor
            ptx::umma_i8(d, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) != 0 ? 1u : 0u);
          ptx::umma_commit<1>(&empty[slot]);
        }
        __syncwarp();
      }
      if (ptx::elect_one()) ptx::umma_commit<1>(&tfull[buf]);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue: fold the limbs
    const int ew = warp & 3;   // a warp may read TMEM lanes 32 (warp % 4) .. + 31
    uint32_t tcount = 0;
    for (int64_t T = blockIdx.x; T < n_tiles; T += gridDim.x, ++tcount) {
      const uint32_t buf = tcount & 1u;
      ptx::mbar_wait(&tfull[buf], (tcount >> 1) & 1u);
      ptx::tc_fence_after();
      uint32_t v[8];
      ptx::tmem_ld8(tmem_base + ((uint32_t)(32 * ew) << 16) + buf * kTcLimbs, v);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
      const int64_t g = T * kTcRows + 32 * ew + lane;
      if (g < n_segs) {
        const int i = owner_of(seg_base, n_inputs, g);
        const int64_t start = offsets[i] + (g - seg_base[i]) * s;
        const int64_t len = min(s, offsets[i + 1] - start);
        if (tc_segment(data, start, len, s, 1)) {
          // sum_n S_n 2^(8n) < 2^31 * 2^57: exact in 128 bits, then 2^64 = 2^3 (mod M)
          unsigned __int128 x = 0;
#pragma unroll
          for (int n = 7; n >= 0; --n) x = (x << 8) + (unsigned __int128)v[n];
          const uint64_t lo = (uint64_t)x, hi = (uint64_t)(x >> 64);
          seg_hash[g] = canon(red((lo & kM) + (lo >> 61) + (hi << 3)));
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<1>(tmem_base, 32);
  }
}

__global__ void phase1_kernel(const uint8_t* __restrict__ data, const int64_t* __restrict__ offsets,
                              const int64_t* __restrict__ seg_base, int32_t n_inputs, int64_t n_segs, int64_t s,
                              Tables tb, uint64_t* __restrict__ seg_hash, int tc_on) {
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
    if (tc_segment(data, start, len, s, tc_on)) continue;   // hashed by phase1_tc_kernel
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
  int32_t num_sms = 148;
  int64_t max_inputs = 0, max_bytes = 0, s = 4096, max_segs = 0;
  uint8_t* d_wgt = nullptr;       // tensor-core limb matrix [s/128][8][128] (null: no TC path)
  int64_t last_segs = 0, last_tc_segs = 0;
  uint8_t* d_stage = nullptr;
  int64_t* d_offsets = nullptr;
  int64_t* d_seg_base = nullptr;
  uint64_t* d_seg_hash = nullptr;
  uint64_t* d_pow16 = nullptr;
  // host staging of the offsets / segment bases, double-buffered so a call never waits
  // for the previous one on the host: slot b = [2 * (max_inputs + 1)] (offsets, seg_base)
  int64_t* h_pinned = nullptr;   // [2 slots][2 * (max_inputs + 1)]
  cudaEvent_t done[2] = {nullptr, nullptr};
  bool pending[2] = {false, false};
  int32_t slot = 0;
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
  cudaFree(h->d_wgt);
  if (h->h_pinned) cudaFreeHost(h->h_pinned);
  for (auto& e : h->done)
    if (e) cudaEventDestroy(e);
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
            cudaMallocHost(&h->h_pinned, 4 * (max_inputs + 1) * sizeof(int64_t)) == cudaSuccess &&
            cudaEventCreateWithFlags(&h->done[0], cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&h->done[1], cudaEventDisableTiming) == cudaSuccess;
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
  if (segment_size % 128 == 0 && segment_size / 128 <= kTcMaxKb) {
    // limb matrix of the tensor-core path: byte k of a segment has weight B^(s-1-k) mod M;
    // limb n of it sits at K-block k/128, row n, 16-B chunk ((k%128)/16) ^ n (128-B swizzle)
    const int64_t n_kb = segment_size / 128;
    std::vector<uint8_t> w((size_t)n_kb * 1024, 0);
    uint64_t wk = 1;   // B^(s-1-k), k from s-1 down
    for (int64_t k = segment_size - 1; k >= 0; --k) {
      const int64_t kb = k / 128, j = k % 128;
      for (int n = 0; n < 8; ++n)
        w[(size_t)kb * 1024 + n * 128 + (((j >> 4) ^ n) << 4) + (j & 15)] = (uint8_t)((wk >> (8 * n)) & 0xFF);
      wk = mulmod_host(wk, kB);
    }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    h->num_sms = nsm;
    if (cudaMalloc(&h->d_wgt, w.size()) != cudaSuccess ||
        cudaMemcpy(h->d_wgt, w.data(), w.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaFuncSetAttribute(phase1_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tc_smem_bytes((int)n_kb)) != cudaSuccess) {
      cudaGetLastError();
      hasher_free(h);
      return AMS_ERR_CUDA;
    }
  }
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
  using namespace ams::hash;
  if (h == nullptr || offsets == nullptr || out_hash == nullptr || n_inputs < 1 || n_inputs > h->max_inputs)
    return AMS_ERR_INVALID_ARGUMENT;
  if (h->broken) return AMS_ERR_CUDA;
  const int64_t total = offsets[n_inputs] - offsets[0];
  if (offsets[0] < 0 || total < 0 || (total > 0 && data == nullptr)) return AMS_ERR_INVALID_ARGUMENT;
  const bool device_data = total > 0 && dev_ptr(data);
  if (total > h->max_bytes) return AMS_ERR_CAPACITY;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaSetDevice(h->device) != cudaSuccess) return AMS_ERR_CUDA;
  // pinned slot b was last read by the call before the previous one (normally long done);
  // the device buffers are ordered after the previous call on the device, not the host
  const int b = h->slot;
  if (h->pending[b] && cudaEventSynchronize(h->done[b]) != cudaSuccess) {
    h->broken = true;
    return AMS_ERR_CUDA;
  }
  h->pending[b] = false;
  if (h->pending[b ^ 1] && cudaStreamWaitEvent(s, h->done[b ^ 1], 0) != cudaSuccess) {
    h->broken = true;
    return AMS_ERR_CUDA;
  }
  int64_t* off = h->h_pinned + (size_t)b * 2 * (h->max_inputs + 1);
  int64_t* base = off + (h->max_inputs + 1);
  int64_t nseg = 0, ntc = 0;
  const uint8_t* src = (total > 0 && !device_data) ? h->d_stage : data;
  // one pass: rebased offsets, monotonicity, segment bases and the tensor-core segment
  // count (shifts for a power-of-two s: this loop is the per-call cost of hashing many
  // tiny actions)
  const int64_t s_len = h->s;
  const bool pow2 = (s_len & (s_len - 1)) == 0;
  const int sh = pow2 ? __builtin_ctzll((unsigned long long)s_len) : 0;
  const int64_t o0 = device_data ? 0 : offsets[0];
  const uintptr_t src_addr = reinterpret_cast<uintptr_t>(src);
  const bool tc = h->d_wgt != nullptr;   // full 16-B aligned segments go to the tensor-core kernel
  int64_t prev = offsets[0];
  for (int32_t i = 0; i < n_inputs; ++i) {
    const int64_t o = prev, o1 = offsets[i + 1];
    if (o1 < o) return AMS_ERR_INVALID_ARGUMENT;
    const int64_t len = o1 - o;
    off[i] = o - o0;
    base[i] = nseg;
    const int64_t full = pow2 ? (len >> sh) : len / s_len;
    nseg += full + ((len - full * s_len) != 0 ? 1 : 0);
    if (tc && ((src_addr + (uintptr_t)(o - o0)) & 15u) == 0) ntc += full;
    prev = o1;
  }
  off[n_inputs] = offsets[n_inputs] - o0;
  base[n_inputs] = nseg;
  if (nseg > h->max_segs) return AMS_ERR_CAPACITY;
  h->last_segs = nseg;
  h->last_tc_segs = ntc;
  bool ok = cudaMemcpyAsync(h->d_offsets, off, (n_inputs + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s) ==
                cudaSuccess &&
            cudaMemcpyAsync(h->d_seg_base, base, (n_inputs + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s) ==
                cudaSuccess;
  if (ok && total > 0 && !device_data)
    ok = cudaMemcpyAsync(h->d_stage, data + offsets[0], total, cudaMemcpyDefault, s) == cudaSuccess;
  if (ok && ntc > 0) {
    const int64_t tiles = (nseg + kTcRows - 1) / kTcRows;
    ams::hash::phase1_tc_kernel<<<(unsigned)std::min<int64_t>(tiles, h->num_sms), kTcThreads,
                                  tc_smem_bytes((int)(h->s / 128)), s>>>(src, h->d_offsets, h->d_seg_base, n_inputs,
                                                                         nseg, h->s, h->d_wgt, h->d_seg_hash);
    ok = cudaGetLastError() == cudaSuccess;
  }
  if (ok && nseg > ntc) {
    const int wpb = 8;
    const int64_t blocks = std::min<int64_t>((nseg + wpb - 1) / wpb, 148 * 16);
    ams::hash::phase1_kernel<<<(unsigned)blocks, wpb * 32, 0, s>>>(src, h->d_offsets, h->d_seg_base, n_inputs, nseg,
                                                                   h->s, h->tb, h->d_seg_hash, ntc > 0 ? 1 : 0);
    ok = cudaGetLastError() == cudaSuccess;
  }
  if (ok) {
    const int wpb = 8;
    ams::hash::phase2_kernel<<<(unsigned)((n_inputs + wpb - 1) / wpb), wpb * 32, 0, s>>>(
        h->d_seg_base, n_inputs, h->d_seg_hash, h->tb, out_hash);
    ok = cudaGetLastError() == cudaSuccess;
  }
  ok = ok && cudaEventRecord(h->done[b], s) == cudaSuccess;
  if (!ok) {
    h->broken = true;
    return AMS_ERR_CUDA;
  }
  h->pending[b] = true;
  h->slot = b ^ 1;
  return AMS_OK;
}

ams_status_t ams_hasher_last_stats(ams_hasher_t h, int64_t* segments, int64_t* tc_segments) {
  if (h == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  if (segments) *segments = h->last_segs;
  if (tc_segments) *tc_segments = h->last_tc_segs;
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
