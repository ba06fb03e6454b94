// ams_exchange.cu -- fused NVLink shard exchange (opt-in).
//
// The default multi-GPU path of ams_match is: intra-GPU merge -> ncclAllGather of each
// rank's [nq][k] list -> G-way merge kernel.  This module replaces the collective with
// direct peer stores over NVLink (CUDA IPC mappings of every rank's receive buffer):
//
//   producer  `merge_push_kernel`: the intra-GPU merge of the partial lists (same code as
//             merge_partials_kernel) stages each query's merged list in shared memory and
//             stores it, coalesced, into EVERY rank's receive buffer slot
//             [parity][rank][q][0..k) (peer pointers; the local one for itself).  Each
//             block then fences at system scope and bumps a local arrival counter; the
//             last block stores `epoch` into its slot of every rank's flag array with a
//             system-scope release.
//   consumer  `merge_wait_kernel`: each block waits (acquire loads) until all G flags of
//             the local array have reached `epoch` (>=: a faster peer may already have
//             raised its flag for e+1), then merges the G received lists by (score desc,
//             global index asc) into the outputs and the hit flags.  The wait is bounded
//             (globaltimer, PeerTable::timeout_ns): on timeout the block writes padding
//             (-1, -inf, miss), sets the pool's error word (host-mapped memory, so the
//             host sees it without a synchronisation) and exits; the next ams_match on
//             that pool returns AMS_ERR_NCCL.
//
// Receive buffers are double-buffered by epoch parity: rank g can only start producing
// call e+2 after its consumer of call e+1 saw rank r's flag for e+1, which rank r raises
// only after it finished consuming call e -- so slot e%2 is never overwritten while read.
// Flags only increase, so a flag at e+1 while rank r still waits for e means peer g's
// slot e%2 holds call e's list (g wrote e+1 into the other parity).
// On one GPU (no peers) `ams_exchange_selftest` runs the same device code for G virtual
// ranks: every producer launch completes before any consumer launch starts, so no kernel
// ever waits on a concurrently running one.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <nccl.h>

#include <cstring>
#include <new>
#include <vector>

#include "ams_internal.cuh"
#include "ams_topk.cuh"

namespace ams {
namespace {

constexpr int kWarpsX = 4;   // queries (warps) per block

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// k rounds of the butterfly arg-max; the merged list lands in the warp's staging area
template <int KT, typename I>
__device__ __forceinline__ void warp_collect(TopK<KT, I>& t, int k, int lane, float* st_s, int64_t* st_i,
                                             int32_t rank, int32_t world, int64_t B, bool to_global) {
  for (int r = 0; r < k; ++r) {
    float bs = t.s[0];
    I bi = t.i[0];
    int bl = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float os = __shfl_xor_sync(0xffffffffu, bs, o);
      const I oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (better(os, oi, bs, bi) || (!better(bs, bi, os, oi) && ol < bl)) {
        bs = os;
        bi = oi;
        bl = ol;
      }
    }
    if (lane == 0) {
      st_s[r] = bi >= 0 ? bs : -CUDART_INF_F;
      st_i[r] = bi >= 0 ? (to_global ? shard_global((int64_t)bi, rank, world, B) : (int64_t)bi) : -1;
    }
    if (lane == bl) t.pop_front();
  }
  __syncwarp();
}

template <int KT>
__global__ void __launch_bounds__(32 * kWarpsX)
    merge_push_kernel(const float* __restrict__ part_s, const int32_t* __restrict__ part_i, int32_t nq, int32_t P,
                      int32_t k, PeerTable peers, unsigned long long epoch, unsigned int* __restrict__ done,
                      int32_t world_for_ids, int64_t B) {
  __shared__ float st_s[kWarpsX][64];
  __shared__ int64_t st_i[kWarpsX][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int q = blockIdx.x * kWarpsX + w;
  const int parity = (int)(epoch & 1ull);
  if (q < nq) {
    TopK<KT, int32_t> t;
    t.init(true);
    for (int p = lane; p < P; p += 32) {
      const int64_t base = ((int64_t)q * P + p) * KT;
      for (int r = 0; r < k; ++r) {
        const int32_t j = part_i[base + r];
        const float v = part_s[base + r];
        if (j < 0 || !better(v, j, t.kth_s, t.kth_i)) break;
        t.insert(v, j, k);
      }
    }
    warp_collect(t, k, lane, st_s[w], st_i[w], peers.rank, world_for_ids, B, world_for_ids > 0);
    // coalesced stores of the k entries into every rank's receive slot
    const int64_t off = (((int64_t)parity * peers.G + peers.rank) * peers.max_q + q) * peers.max_k;
    for (int g = 0; g < peers.G; ++g)
      for (int r = lane; r < k; r += 32) {
        peers.s[g][off + r] = st_s[w][r];
        peers.i[g][off + r] = st_i[w][r];
      }
  }
  __threadfence_system();   // every thread: its peer stores are visible system-wide first
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicInc(done, gridDim.x - 1) == gridDim.x - 1) {    // last block of this rank
      __threadfence_system();
      for (int g = 0; g < peers.G; ++g) st_release_sys(peers.flag[g] + peers.rank, epoch);
    }
  }
}

template <int KT>
__global__ void __launch_bounds__(32 * kWarpsX)
    merge_wait_kernel(PeerTable peers, int32_t nq, int32_t k, unsigned long long epoch, float* __restrict__ out_s,
                      int64_t* __restrict__ out_i, uint8_t* __restrict__ out_hit, float threshold) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ int timed_out;
  if (threadIdx.x == 0) timed_out = 0;
  __syncthreads();
  if (threadIdx.x < peers.G) {
    const unsigned long long* f = peers.flag[peers.rank] + threadIdx.x;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(f) < epoch) {
      if (globaltimer_ns() - t0 > peers.timeout_ns) {
        atomicExch(&timed_out, 1);
        atomicOr(peers.err, 1u);   // host-mapped: visible to the host without a sync
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
  const int q = blockIdx.x * kWarpsX + w;
  if (q >= nq) return;
  if (timed_out) {   // a peer never delivered this epoch: padding, miss
    for (int r = lane; r < k; r += 32) {
      out_s[(int64_t)q * k + r] = -CUDART_INF_F;
      out_i[(int64_t)q * k + r] = -1;
    }
    if (lane == 0) out_hit[q] = 0;
    return;
  }
  const int parity = (int)(epoch & 1ull);
  const float* rs = peers.s[peers.rank];
  const int64_t* ri = peers.i[peers.rank];
  TopK<KT, int64_t> t;
  t.init(true);
  for (int g = lane; g < peers.G; g += 32) {
    const int64_t base = (((int64_t)parity * peers.G + g) * peers.max_q + q) * peers.max_k;
    for (int r = 0; r < k; ++r) {
      const int64_t j = ri[base + r];
      const float v = rs[base + r];
      if (j < 0 || !better(v, j, t.kth_s, t.kth_i)) break;
      t.insert(v, j, k);
    }
  }
  float s0 = -CUDART_INF_F;
  int64_t i0 = -1;
  for (int r = 0; r < k; ++r) {
    float bs = t.s[0];
    int64_t bi = t.i[0];
    int bl = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float os = __shfl_xor_sync(0xffffffffu, bs, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (better(os, oi, bs, bi) || (!better(bs, bi, os, oi) && ol < bl)) {
        bs = os;
        bi = oi;
        bl = ol;
      }
    }
    if (lane == 0) {
      out_s[(int64_t)q * k + r] = bi >= 0 ? bs : -CUDART_INF_F;
      out_i[(int64_t)q * k + r] = bi;
    }
    if (r == 0) {
      s0 = bs;
      i0 = bi;
    }
    if (lane == bl) t.pop_front();
  }
  if (lane == 0) out_hit[q] = (i0 >= 0 && s0 >= threshold) ? 1 : 0;
}

// lists [nq][k] -> partial-list layout [nq][1][KT] with (-inf, -1) padding (self-test input)
__global__ void to_partials_kernel(const float* __restrict__ s, const int64_t* __restrict__ i, int32_t nq, int32_t k,
                                   int32_t KT, float* __restrict__ ps, int32_t* __restrict__ pi) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nq * KT) return;
  const int64_t q = e / KT, r = e % KT;
  ps[e] = r < k ? s[q * k + r] : -CUDART_INF_F;
  pi[e] = r < k ? (int32_t)i[q * k + r] : -1;
}

template <int KT>
cudaError_t launch_push(const float* ps, const int32_t* pi, int32_t nq, int32_t P, int32_t k, const PeerTable& pt,
                        unsigned long long epoch, unsigned int* done, int32_t world_ids, int64_t B, cudaStream_t s) {
  merge_push_kernel<KT><<<(nq + kWarpsX - 1) / kWarpsX, 32 * kWarpsX, 0, s>>>(ps, pi, nq, P, k, pt, epoch, done,
                                                                              world_ids, B);
  return cudaGetLastError();
}
template <int KT>
cudaError_t launch_wait(const PeerTable& pt, int32_t nq, int32_t k, unsigned long long epoch, float* os, int64_t* oi,
                        uint8_t* oh, float th, cudaStream_t s) {
  merge_wait_kernel<KT><<<(nq + kWarpsX - 1) / kWarpsX, 32 * kWarpsX, 0, s>>>(pt, nq, k, epoch, os, oi, oh, th);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_exchange_push(int KT, const float* ps, const int32_t* pi, int32_t nq, int32_t P, int32_t k,
                                 const PeerTable& pt, unsigned long long epoch, unsigned int* done, int32_t world_ids,
                                 int64_t B, cudaStream_t s) {
  switch (KT) {
    case 8: return launch_push<8>(ps, pi, nq, P, k, pt, epoch, done, world_ids, B, s);
    case 16: return launch_push<16>(ps, pi, nq, P, k, pt, epoch, done, world_ids, B, s);
    case 32: return launch_push<32>(ps, pi, nq, P, k, pt, epoch, done, world_ids, B, s);
    default: return launch_push<64>(ps, pi, nq, P, k, pt, epoch, done, world_ids, B, s);
  }
}

cudaError_t launch_exchange_wait(int KT, const PeerTable& pt, int32_t nq, int32_t k, unsigned long long epoch,
                                 float* os, int64_t* oi, uint8_t* oh, float th, cudaStream_t s) {
  switch (KT) {
    case 8: return launch_wait<8>(pt, nq, k, epoch, os, oi, oh, th, s);
    case 16: return launch_wait<16>(pt, nq, k, epoch, os, oi, oh, th, s);
    case 32: return launch_wait<32>(pt, nq, k, epoch, os, oi, oh, th, s);
    default: return launch_wait<64>(pt, nq, k, epoch, os, oi, oh, th, s);
  }
}

cudaError_t launch_to_partials(const float* s, const int64_t* i, int32_t nq, int32_t k, int32_t KT, float* ps,
                               int32_t* pi, cudaStream_t st) {
  const int64_t n = (int64_t)nq * KT;
  to_partials_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s, i, nq, k, KT, ps, pi);
  return cudaGetLastError();
}

}  // namespace ams

extern "C" {

ams_status_t ams_exchange_selftest(int32_t G, int32_t nq, int32_t k, int32_t rounds, float threshold,
                                   const float* in_score, const int64_t* in_index, float* out_score,
                                   int64_t* out_index, uint8_t* out_hit, int32_t flags, void* stream) {
  using namespace ams;
  if (G < 1 || G > kMaxPeers || nq < 1 || k < 1 || k > 64 || rounds < 1 || in_score == nullptr ||
      in_index == nullptr || out_score == nullptr || out_index == nullptr || out_hit == nullptr ||
      (flags & ~(AMS_SELFTEST_LATE_CONSUMER | AMS_SELFTEST_DROP_LAST)) != 0 ||
      ((flags & AMS_SELFTEST_LATE_CONSUMER) && G < 2))
    return AMS_ERR_INVALID_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int KT = pick_KT(k);
  const size_t slot = (size_t)2 * G * nq * k;
  std::vector<void*> allocs;
  auto dalloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return p;
  };
  ams_status_t st = AMS_OK;
  PeerTable base{};
  base.G = G;
  base.max_q = nq;
  base.max_k = k;
  // the drop test must end quickly; otherwise the library's bound
  base.timeout_ns = (flags & AMS_SELFTEST_DROP_LAST) ? 20ull * 1000 * 1000 : kPeerTimeoutNs;
  unsigned int* err_host = nullptr;
  if (cudaHostAlloc((void**)&err_host, sizeof(unsigned int), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&base.err, err_host, 0) != cudaSuccess) {
    cudaGetLastError();
    if (err_host) cudaFreeHost(err_host);
    return AMS_ERR_CUDA;
  }
  *err_host = 0;
  std::vector<unsigned int*> done(G);
  for (int g = 0; g < G && st == AMS_OK; ++g) {
    base.s[g] = static_cast<float*>(dalloc(slot * 4));
    base.i[g] = static_cast<int64_t*>(dalloc(slot * 8));
    base.flag[g] = static_cast<unsigned long long*>(dalloc(G * 8));
    done[g] = static_cast<unsigned int*>(dalloc(4));
    if (!base.s[g] || !base.i[g] || !base.flag[g] || !done[g]) st = AMS_ERR_OUT_OF_MEMORY;
    else if (cudaMemsetAsync(base.flag[g], 0, G * 8, s) != cudaSuccess || cudaMemsetAsync(done[g], 0, 4, s) != cudaSuccess)
      st = AMS_ERR_CUDA;
  }
  float* ps = static_cast<float*>(dalloc((size_t)G * nq * KT * 4));
  int32_t* pi = static_cast<int32_t*>(dalloc((size_t)G * nq * KT * 4));
  if (st == AMS_OK && (!ps || !pi)) st = AMS_ERR_OUT_OF_MEMORY;
  auto push = [&](int g, int rd) {
    if (st != AMS_OK) return;
    const unsigned long long epoch = (unsigned long long)rd + 1;
    const float* in_s = in_score + ((size_t)rd * G + g) * nq * k;
    const int64_t* in_i = in_index + ((size_t)rd * G + g) * nq * k;
    if (launch_to_partials(in_s, in_i, nq, k, KT, ps + (size_t)g * nq * KT, pi + (size_t)g * nq * KT, s) !=
        cudaSuccess)
      st = AMS_ERR_CUDA;
    PeerTable pt = base;
    pt.rank = g;
    // ids are already global (world_ids = 0: no shard map)
    if (st == AMS_OK && launch_exchange_push(KT, ps + (size_t)g * nq * KT, pi + (size_t)g * nq * KT, nq, 1, k, pt,
                                             epoch, done[g], 0, 0, s) != cudaSuccess)
      st = AMS_ERR_CUDA;
  };
  auto wait = [&](int g, int rd) {
    if (st != AMS_OK) return;
    PeerTable pt = base;
    pt.rank = g;
    const size_t o = ((size_t)rd * G + g) * nq;
    if (launch_exchange_wait(KT, pt, nq, k, (unsigned long long)rd + 1, out_score + o * k, out_index + o * k,
                             out_hit + o, threshold, s) != cudaSuccess)
      st = AMS_ERR_CUDA;
  };
  // Every consumer is enqueued after the producers it waits for (no kernel ever waits on a
  // concurrently running one).  LATE_CONSUMER: rank G-1 consumes round rd-1 only after the
  // other ranks already produced round rd (their flags are then ahead of the epoch it waits
  // for -- the order a descheduled host thread produces on a real box).  DROP_LAST: rank
  // G-1 never produces the last round; its consumers must time out, not hang.
  const bool late = (flags & AMS_SELFTEST_LATE_CONSUMER) != 0;
  const bool drop = (flags & AMS_SELFTEST_DROP_LAST) != 0;
  for (int rd = 0; rd < rounds && st == AMS_OK; ++rd) {
    const bool skip_last = drop && rd == rounds - 1;
    for (int g = 0; g < G - 1; ++g) push(g, rd);
    if (late && rd > 0) wait(G - 1, rd - 1);
    if (!skip_last) push(G - 1, rd);
    for (int g = 0; g < G - 1; ++g) wait(g, rd);
    if (!late) wait(G - 1, rd);
  }
  if (late) wait(G - 1, rounds - 1);
  if (cudaStreamSynchronize(s) != cudaSuccess) st = AMS_ERR_CUDA;
  if (st == AMS_OK && *err_host != 0) st = AMS_ERR_NCCL;   // a wait timed out
  for (void* p : allocs) cudaFree(p);
  cudaFreeHost(err_host);
  return st;
}

}  // extern "C"
