// ams_kernels.cu -- record (append), query prep, the exact fp32 SIMT matcher and the
// k-way merges of AMS action-context matching (3.2.1).
#include <cuda_bf16.h>
#include <math_constants.h>

#include "ams_internal.cuh"
#include "ams_ptx.cuh"
#include "ams_topk.cuh"

namespace ams {

namespace {

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------------
// Record ("adds the unseen vector ... into the context pool").
// One warp per source row; the rank keeps only the rows its shard map owns.
// bf16: inv_norm = fp32(1 / sqrt(sum x^2 in fp64)) over the STORED values.
// fp32: canonical ss = fmaf(x_t, x_t, ss), t ascending; inv = 1.0f / sqrtf(ss).
// ---------------------------------------------------------------------------------
template <bool BF16>
__global__ void append_kernel(const void* __restrict__ src, const float* __restrict__ jsrc, int64_t n,
                              int64_t first_global, int32_t d, int32_t J, int32_t JP, int32_t rank,
                              int32_t world, int64_t B, void* __restrict__ emb, float* __restrict__ inv_norm,
                              float* __restrict__ joints) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  const int64_t o = first_global + r;
  if (shard_owner(o, world, B) != rank) return;
  const int64_t l = shard_local(o, world, B);
  if (BF16) {
    const uint4* s4 = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(src) + r * d);
    uint4* d4 = reinterpret_cast<uint4*>(static_cast<uint16_t*>(emb) + l * d);
    double ss = 0.0;
    for (int c = lane; c < d / 8; c += 32) {
      const uint4 w = s4[c];
      d4[c] = w;
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double a = bf16_lo(ws[q]), b = bf16_hi(ws[q]);
        ss += a * a;
        ss += b * b;
      }
    }
    ss = warp_sum_f64(ss);
    if (lane == 0) inv_norm[l] = ss > 0.0 ? __double2float_rn(1.0 / sqrt(ss)) : 0.0f;
  } else {
    const float* s = static_cast<const float*>(src) + r * d;
    float* e = static_cast<float*>(emb) + l * d;
    for (int c = lane; c < d; c += 32) e[c] = s[c];
    if (lane == 0) {
      float ss = 0.0f;
      for (int t = 0; t < d; ++t) ss = __fmaf_rn(s[t], s[t], ss);
      inv_norm[l] = ss > 0.0f ? __fdiv_rn(1.0f, __fsqrt_rn(ss)) : 0.0f;
    }
  }
  if (lane < JP) joints[joint_offset(l, lane, JP)] = lane < J ? jsrc[r * J + lane] : 0.0f;
}

// ---------------------------------------------------------------------------------
// Query prep: stage the query rows, inv_q, zero-padded joints.  One warp per query.
// ---------------------------------------------------------------------------------
// Staged row q holds the caller's query perm[q] (perm == nullptr: identity).
constexpr int kPrepWarps = 8;   // queries (warps) per query_prep block

template <bool BF16>
__global__ void query_prep_kernel(const void* __restrict__ src, const float* __restrict__ jsrc, int32_t nq,
                                  int32_t d, int32_t J, int32_t JP, const int32_t* __restrict__ perm,
                                  void* __restrict__ q_stage, float* __restrict__ q_inv,
                                  float* __restrict__ q_joints, uint32_t* __restrict__ zero_a, int32_t n_zero_a,
                                  uint32_t* __restrict__ zero_b, int32_t n_zero_b) {
  // the dense kernel that follows (launched as a programmatic dependent) may start its
  // prologue now; it reads nothing of ours before griddep_wait()
  ptx::griddep_launch_dependents();
  {   // its counters (per-query bounds and union slots, or candidate counts) start at zero
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
    for (int i = gt; i < n_zero_a; i += gs) zero_a[i] = 0u;
    for (int i = gt; i < n_zero_b; i += gs) zero_b[i] = 0u;
  }
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const int64_t o = perm != nullptr ? (int64_t)perm[q] : (int64_t)q;
  if constexpr (BF16) {
    const uint4* s4 = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(src) + o * d);
    uint4* d4 = reinterpret_cast<uint4*>(static_cast<uint16_t*>(q_stage) + (int64_t)q * d);
    double ss = 0.0;
    // 4 pieces per lane in flight before any store (s4 may alias d4 as far as the compiler
    // knows, which would otherwise serialise every load behind the previous store)
    for (int c0 = 0; c0 < d / 8; c0 += 128) {
      uint4 wv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + 32 * u + lane;
        wv[u] = c < d / 8 ? __ldg(s4 + c) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + 32 * u + lane;
        if (c >= d / 8) continue;
        if (s4 != d4) d4[c] = wv[u];
        const uint32_t ws[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double a = bf16_lo(ws[k]), b = bf16_hi(ws[k]);
          ss += a * a;
          ss += b * b;
        }
      }
    }
    ss = warp_sum_f64(ss);
    if (lane == 0) q_inv[q] = ss > 0.0 ? __double2float_rn(1.0 / sqrt(ss)) : 0.0f;
  } else {
    // the warp stages the query through shared memory in coalesced 1024-value chunks (and
    // copies it to q_stage); lane 0 runs the canonical chain (t ascending, one fmaf chain)
    // from shared memory -- one memory round trip per chunk instead of one per few values
    __shared__ __align__(16) float qbuf[kPrepWarps][1024];
    const float* s = static_cast<const float*>(src) + o * d;
    float* e = static_cast<float*>(q_stage) + (int64_t)q * d;
    float* buf = qbuf[threadIdx.x >> 5];
    float ss = 0.0f;
    for (int c0 = 0; c0 < d; c0 += 1024) {
      const int n = min(1024, d - c0);   // a multiple of 32 (d % 64 == 0)
      __syncwarp();
      float v[32];   // all of the lane's loads in flight before any store (see the bf16 branch)
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = 32 * u < n ? __ldg(s + c0 + 32 * u + lane) : 0.0f;
#pragma unroll
      for (int u = 0; u < 32; ++u)
        if (32 * u < n) {
          buf[32 * u + lane] = v[u];
          if (s != e) e[c0 + 32 * u + lane] = v[u];
        }
      __syncwarp();
      if (lane == 0) {   // n % 4 == 0 (d % 64 == 0); 16-byte shared loads, several in flight
        const float4* b4 = reinterpret_cast<const float4*>(buf);
#pragma unroll 8
        for (int t4 = 0; t4 < n / 4; ++t4) {
          const float4 v = b4[t4];
          ss = __fmaf_rn(v.x, v.x, ss);
          ss = __fmaf_rn(v.y, v.y, ss);
          ss = __fmaf_rn(v.z, v.z, ss);
          ss = __fmaf_rn(v.w, v.w, ss);
        }
      }
    }
    if (lane == 0) q_inv[q] = ss > 0.0f ? __fdiv_rn(1.0f, __fsqrt_rn(ss)) : 0.0f;
  }
  if (lane < JP) q_joints[(int64_t)q * JP + lane] = lane < J ? jsrc[o * J + lane] : 0.0f;
}

// ---------------------------------------------------------------------------------
// Query order for gated batches: a counting sort of the queries by a two-joint key
// (one block).  Any order gives the same results (every query is scored
// independently); this one makes the 32 queries of a warp span a small box in
// (joint 0, joint 1), so most pool rows fail the warp-level gate test of the epilogue
// (ams_match_tc.cu epi_chunk_sorted) and of gate_scan_kernel.  Key = b0 * B1 + b1 with
// b0 a linear bin of joint 0 among B0 = clamp(nq / 256, 1, 64) bins (~256 queries, i.e.
// 8 warps, per b0 bin) and b1 a linear bin of joint 1 among B1 = 4096 / B0 bins, each
// between the batch's min and max (J = 1: joint 0 alone, 4096 bins).  Order within a
// bin is arbitrary.
// ---------------------------------------------------------------------------------
constexpr int kOrderBins = 4096;
constexpr int kOrderThreads = 1024;

__device__ __forceinline__ void block_minmax(float& lo, float& hi, float* red_lo, float* red_hi) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __syncthreads();
  if (lane == 0) {
    red_lo[w] = lo;
    red_hi[w] = hi;
  }
  __syncthreads();
  lo = red_lo[0];
  hi = red_hi[0];
  for (int i = 1; i < kOrderThreads / 32; ++i) {
    lo = fminf(lo, red_lo[i]);
    hi = fmaxf(hi, red_hi[i]);
  }
}

// linear bin of v among n bins of [lo, hi] (NaN and out-of-range values clamp)
__device__ __forceinline__ int lin_bin(float v, float lo, float scale, int n) {
  const float f = (v - lo) * scale;
  return (f >= 0.0f && f < (float)n) ? (int)f : (f >= 0.0f ? n - 1 : 0);
}

__global__ void __launch_bounds__(kOrderThreads)
    query_order_kernel(const float* __restrict__ jsrc, int32_t J, int32_t nq, int32_t* __restrict__ perm) {
  __shared__ uint32_t hist[kOrderBins];
  __shared__ float red_lo[kOrderThreads / 32], red_hi[kOrderThreads / 32];
  __shared__ uint32_t wsum[kOrderThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nj = J >= 2 ? 2 : 1;
  const int B0 = nj == 1 ? kOrderBins : max(1, min(64, nq / 256));
  const int B1 = kOrderBins / B0;
  float lo[2], sc[2];
  for (int t = 0; t < nj; ++t) {
    float l = CUDART_INF_F, h = -CUDART_INF_F;
    for (int q = tid; q < nq; q += kOrderThreads) {
      const float v = jsrc[(int64_t)q * J + t];
      if (v == v) {
        l = fminf(l, v);
        h = fmaxf(h, v);
      }
    }
    block_minmax(l, h, red_lo, red_hi);
    const float span = h - l;
    lo[t] = l;
    sc[t] = (span > 1e-30f && span < CUDART_INF_F) ? (float)(t == 0 ? B0 : B1) / span : 0.0f;
  }
  auto key_of = [&](int q) -> int {
    const int b0 = lin_bin(jsrc[(int64_t)q * J], lo[0], sc[0], B0);
    return nj == 1 ? b0 : b0 * B1 + lin_bin(jsrc[(int64_t)q * J + 1], lo[1], sc[1], B1);
  };
  for (int b = tid; b < kOrderBins; b += kOrderThreads) hist[b] = 0u;
  __syncthreads();
  for (int q = tid; q < nq; q += kOrderThreads) atomicAdd(&hist[key_of(q)], 1u);
  __syncthreads();
  // exclusive scan: thread t owns bins [4t, 4t+4)
  constexpr int per = kOrderBins / kOrderThreads;
  uint32_t v[per], run = 0;
#pragma unroll
  for (int i = 0; i < per; ++i) {
    v[i] = hist[tid * per + i];
    run += v[i];
  }
  uint32_t incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t base = 0;
  for (int i = 0; i < w; ++i) base += wsum[i];
  base += incl - run;
#pragma unroll
  for (int i = 0; i < per; ++i) {
    hist[tid * per + i] = base;
    base += v[i];
  }
  __syncthreads();
  for (int q = tid; q < nq; q += kOrderThreads) {
    const uint32_t pos = atomicAdd(&hist[key_of(q)], 1u);
    perm[pos] = q;
  }
}

// ---------------------------------------------------------------------------------
// Exact fp32 matcher (the bit-exact config, BASELINE.json configs[0]).
// Block = (query, row split); thread t scans rows lo+t, lo+t+128, ... in increasing
// order: canonical gate (fp32 RN sub, fmaf chain), canonical dot (fmaf chain, t
// ascending), s = (acc * inv_q) * inv_e; running top-k in registers.  Partial list
// p = split * 128 + t of query q lands at part[(q * P + p) * KT].
// ---------------------------------------------------------------------------------
constexpr int kSimtChunk = 1024;   // floats of a pool row staged per round trip (4 KB per warp)

template <int KT>
__global__ void __launch_bounds__(kSimtThreads)
    match_simt_f32_kernel(const float* __restrict__ emb, const float* __restrict__ inv_e,
                          const float* __restrict__ pj, int64_t L, const float* __restrict__ q,
                          const float* __restrict__ inv_q, const float* __restrict__ qj, int32_t d, int32_t JP,
                          int32_t S, int32_t k, float g2, int32_t gated, float* __restrict__ part_s,
                          int32_t* __restrict__ part_i, int32_t P) {
  extern __shared__ __align__(16) float qs[];
  ptx::griddep_wait();   // a programmatic dependent of the query prep
  const int qi = blockIdx.x / S;
  const int sp = blockIdx.x % S;
  for (int t = threadIdx.x; t < d; t += blockDim.x) qs[t] = q[(int64_t)qi * d + t];
  float r[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) r[t] = t < JP ? qj[(int64_t)qi * JP + t] : 0.0f;
  const float iq = inv_q[qi];
  __syncthreads();
  const int64_t lo = L * sp / S, hi = L * (sp + 1) / S;
  TopK<KT, int32_t> top;
  top.init(true);
  // Rows are walked warp-synchronously (lane = row); the rows of a step that pass the gate
  // are scored one at a time: the warp stages the row through its shared-memory buffer
  // in coalesced 16-byte pieces (one memory round trip per kSimtChunk values instead of
  // one per few values of a lone thread's loads), then the owning lane runs the canonical
  // chain from shared memory (acc = fmaf(q_t, e_t, acc), t ascending -- the oracle's order).
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* rowbuf = qs + ((d + 3) & ~3) + w * kSimtChunk;   // [warps][kSimtChunk]
  for (int64_t jb = lo + (threadIdx.x & ~31); jb < hi; jb += blockDim.x) {
    const int64_t j = jb + lane;
    bool ok = j < hi;
    if (ok && gated) {
      float ds = 0.0f;
#pragma unroll
      for (int t = 0; t < 16; ++t)
        if (t < JP) {
          const float df = __fsub_rn(r[t], pj[joint_offset(j, t, JP)]);
          ds = __fmaf_rn(df, df, ds);
        }
      ok = ds <= g2;
    }
    uint32_t m = __ballot_sync(0xffffffffu, ok);
    while (m != 0u) {
      const int src = __ffs(m) - 1;
      m &= m - 1u;
      const int64_t jr = jb + src;
      const float4* e4 = reinterpret_cast<const float4*>(emb + jr * d);   // rows 16-B aligned: d % 64 == 0
      float acc = 0.0f;
      for (int c0 = 0; c0 < d; c0 += kSimtChunk) {
        const int n4 = min(kSimtChunk, d - c0) / 4;
        __syncwarp();
        for (int i = lane; i < n4; i += 32) reinterpret_cast<float4*>(rowbuf)[i] = __ldg(e4 + c0 / 4 + i);
        __syncwarp();
        if (lane == src) {
          const float4* q4 = reinterpret_cast<const float4*>(qs + c0);
          const float4* r4 = reinterpret_cast<const float4*>(rowbuf);
#pragma unroll 4
          for (int t4 = 0; t4 < n4; ++t4) {
            const float4 ev = r4[t4], qv = q4[t4];
            acc = __fmaf_rn(qv.x, ev.x, acc);
            acc = __fmaf_rn(qv.y, ev.y, acc);
            acc = __fmaf_rn(qv.z, ev.z, acc);
            acc = __fmaf_rn(qv.w, ev.w, acc);
          }
        }
      }
      if (lane == src) {
        const float sc = __fmul_rn(__fmul_rn(acc, iq), inv_e[jr]);
        if (sc > top.kth_s) top.insert_monotone(sc, (int32_t)jr, k);
      }
    }
  }
  const int64_t base = ((int64_t)qi * P + (int64_t)sp * blockDim.x + threadIdx.x) * KT;
#pragma unroll
  for (int t = 0; t < KT; ++t) {
    part_s[base + t] = top.s[t];
    part_i[base + t] = top.i[t];
  }
}

// ---------------------------------------------------------------------------------
// fp32 exact matcher for UNGATED calls (configs[0]'s "plus an ungated run"): every pair is
// scored, so the thread-per-row kernel above (one dependent 512-long fmaf chain per pair
// per thread, uncoalesced row reads) is latency-bound.  Here a block owns a tile of
// kTileRows rows x kTileQ queries; K advances in chunks of kTileK staged transposed in
// shared memory; each thread runs 2 x 2 independent canonical chains (acc = fmaf(q_t, e_t,
// acc), t ascending -- exactly the oracle's order), then s = RN(RN(acc * iq) * ie).  One
// thread per query inserts the tile's kTileRows scores in row order (insert_monotone keeps
// the lowest index first among ties) and writes the tile's list: partial list p = row
// tile of query q at part[(q * P + p) * KT], P = ceil(L / kTileRows).
// ---------------------------------------------------------------------------------
constexpr int kTileRows = 32, kTileQ = 16, kTileK = 64;
constexpr int kTileThreads = (kTileRows / 2) * (kTileQ / 2);   // 128

template <int KT>
__global__ void __launch_bounds__(kTileThreads)
    match_f32_tile_kernel(const float* __restrict__ emb, const float* __restrict__ inv_e, int64_t L,
                          const float* __restrict__ q, const float* __restrict__ inv_q, int32_t nq, int32_t d,
                          int32_t k, float* __restrict__ part_s, int32_t* __restrict__ part_i, int32_t P) {
  __shared__ float sR[kTileK][kTileRows + 1];
  __shared__ float sQ[kTileK][kTileQ + 1];
  __shared__ float sS[kTileQ][kTileRows + 1];
  ptx::griddep_wait();   // a programmatic dependent of the query prep
  const int rt = blockIdx.x, qt = blockIdx.y;
  const int64_t r0 = (int64_t)rt * kTileRows;
  const int q0 = qt * kTileQ;
  const int tid = threadIdx.x;
  const int rg = tid % (kTileRows / 2), qg = tid / (kTileRows / 2);   // rows 2rg, 2rg+1; queries 2qg, 2qg+1
  float acc[2][2] = {{0.0f, 0.0f}, {0.0f, 0.0f}};
  for (int t0 = 0; t0 < d; t0 += kTileK) {
    __syncthreads();
    for (int i = tid; i < kTileRows * kTileK; i += kTileThreads) {   // coalesced along t
      const int r = i / kTileK, t = i % kTileK;
      sR[t][r] = (r0 + r < L) ? emb[(r0 + r) * d + t0 + t] : 0.0f;
    }
    for (int i = tid; i < kTileQ * kTileK; i += kTileThreads) {
      const int c = i / kTileK, t = i % kTileK;
      sQ[t][c] = (q0 + c < nq) ? q[(int64_t)(q0 + c) * d + t0 + t] : 0.0f;
    }
    __syncthreads();
#pragma unroll 8
    for (int t = 0; t < kTileK; ++t) {
      const float e0 = sR[t][2 * rg], e1 = sR[t][2 * rg + 1];
      const float a0 = sQ[t][2 * qg], a1 = sQ[t][2 * qg + 1];
      acc[0][0] = __fmaf_rn(a0, e0, acc[0][0]);
      acc[0][1] = __fmaf_rn(a1, e0, acc[0][1]);
      acc[1][0] = __fmaf_rn(a0, e1, acc[1][0]);
      acc[1][1] = __fmaf_rn(a1, e1, acc[1][1]);
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t j = r0 + 2 * rg + i;
      const int qi = q0 + 2 * qg + c;
      const float s = (j < L && qi < nq) ? __fmul_rn(__fmul_rn(acc[i][c], inv_q[qi]), inv_e[j]) : -CUDART_INF_F;
      sS[2 * qg + c][2 * rg + i] = s;
    }
  __syncthreads();
  if (tid < kTileQ && q0 + tid < nq) {
    TopK<KT, int32_t> top;
    top.init(true);
    for (int r = 0; r < kTileRows; ++r) {
      const float s = sS[tid][r];
      if (r0 + r < L && s > top.kth_s) top.insert_monotone(s, (int32_t)(r0 + r), k);
    }
    const int64_t base = ((int64_t)(q0 + tid) * P + rt) * KT;
#pragma unroll
    for (int r = 0; r < KT; ++r) {
      part_s[base + r] = top.s[r];
      part_i[base + r] = top.i[r];
    }
  }
}

// ---------------------------------------------------------------------------------
// Warp-cooperative k-way merge: lanes build register top-k lists from a strided subset
// of the input lists (sorted lists: stop at the first entry that cannot enter), then k
// rounds of a butterfly arg-max by (score desc, index asc) emit the merged list.
// ---------------------------------------------------------------------------------
template <int KT, typename I>
__device__ __forceinline__ void warp_emit(TopK<KT, I>& t, int k, int lane, float* out_s, int64_t* out_i,
                                         uint8_t* out_hit, float threshold, int32_t rank, int32_t world,
                                         int64_t B, bool to_global) {
  float s0 = -CUDART_INF_F;
  int64_t i0 = -1;
  for (int r = 0; r < k; ++r) {
    if (!__any_sync(0xffffffffu, t.i[0] >= 0)) {   // every list exhausted: pad the rest
      for (int rr = r + lane; rr < k; rr += 32) {
        out_s[rr] = -CUDART_INF_F;
        out_i[rr] = -1;
      }
      break;
    }
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
    int64_t gi = -1;
    if (bi >= 0) gi = to_global ? shard_global((int64_t)bi, rank, world, B) : (int64_t)bi;
    if (lane == 0) {
      out_s[r] = bi >= 0 ? bs : -CUDART_INF_F;
      out_i[r] = gi;
    }
    if (r == 0) {
      s0 = bs;
      i0 = gi;
    }
    if (lane == bl) t.pop_front();
  }
  if (out_hit != nullptr && lane == 0) *out_hit = (i0 >= 0 && s0 >= threshold) ? 1 : 0;
}

// Lower bound of query q's k-th best score left by the tcgen05 kernel (ordered-u32, 0 =
// none): the max over lists of their KT-th best, and -- when every one of the k union
// slots is filled -- the minimum slot (k distinct rows score at least that much).  Rows
// scoring below it cannot be among the k best; equal scores are kept for the tie rule.
__device__ __forceinline__ float tc_lower_bound(const uint32_t* __restrict__ bound, const uint32_t* __restrict__ slots,
                                                int32_t slot_stride, int32_t k, int q) {
  float b = -CUDART_INF_F;
  if (bound != nullptr) {
    const uint32_t u = bound[q];
    if (u != 0u) b = ptx::ord2f(u);
  }
  if (slots != nullptr) {
    uint32_t mn = 0xFFFFFFFFu;
    for (int r = 0; r < k; ++r) mn = min(mn, slots[(int64_t)q * slot_stride + r]);
    if (mn != 0u) b = fmaxf(b, ptx::ord2f(mn));
  }
  return b;
}

// One query's P partial lists into lane-held TopK lists: lanes take lists lane, lane +
// stride, ... (heads loaded kHeads at a time so their loads are in flight together) and
// walk each sorted list while its entries can still enter (>= lb, better than the lane's
// KT-th).
template <int KT>
__device__ __forceinline__ void gather_lists(const float* __restrict__ part_s, const int32_t* __restrict__ part_i,
                                             int q, int32_t P, int32_t k, float lb, int first, int stride,
                                             TopK<KT, int32_t>& t) {
  constexpr int kHeads = 8;
  for (int p0 = first; p0 < P; p0 += stride * kHeads) {
    float hs[kHeads];
    int32_t hj[kHeads];
#pragma unroll
    for (int u = 0; u < kHeads; ++u) {
      const int p = p0 + u * stride;
      hj[u] = -1;
      hs[u] = -CUDART_INF_F;
      if (p < P) {
        const int64_t base = ((int64_t)q * P + p) * KT;
        hj[u] = part_i[base];
        hs[u] = part_s[base];
      }
    }
#pragma unroll
    for (int u = 0; u < kHeads; ++u) {
      if (hj[u] < 0 || hs[u] < lb || !better(hs[u], hj[u], t.kth_s, t.kth_i)) continue;
      t.insert(hs[u], hj[u], k);
      const int64_t base = ((int64_t)q * P + p0 + u * stride) * KT;
      if constexpr (KT <= 16) {
        // the rest of the list in one round of 16-B loads (not one dependent load per entry)
        float vs[KT];
        int32_t vj[KT];
#pragma unroll
        for (int r = 0; r < KT; r += 4) {
          const float4 a = *reinterpret_cast<const float4*>(part_s + base + r);
          const int4 b = *reinterpret_cast<const int4*>(part_i + base + r);
          vs[r] = a.x, vs[r + 1] = a.y, vs[r + 2] = a.z, vs[r + 3] = a.w;
          vj[r] = b.x, vj[r + 1] = b.y, vj[r + 2] = b.z, vj[r + 3] = b.w;
        }
#pragma unroll
        for (int r = 1; r < KT; ++r) {
          if (r >= k || vj[r] < 0 || vs[r] < lb || !better(vs[r], vj[r], t.kth_s, t.kth_i)) break;
          t.insert(vs[r], vj[r], k);
        }
      } else {   // long lists: registers would spill; walk entry by entry
        for (int r = 1; r < k; ++r) {
          const int32_t j = part_i[base + r];
          const float v = part_s[base + r];
          if (j < 0 || v < lb || !better(v, j, t.kth_s, t.kth_i)) break;
          t.insert(v, j, k);
        }
      }
    }
  }
}

template <int KT>
__global__ void merge_partials_kernel(const float* __restrict__ part_s, const int32_t* __restrict__ part_i,
                                      int32_t nq, int32_t P, int32_t k, float* __restrict__ out_s,
                                      int64_t* __restrict__ out_i, uint8_t* __restrict__ out_hit,
                                      float threshold, int32_t rank, int32_t world, int64_t B,
                                      const uint32_t* __restrict__ bound, const uint32_t* __restrict__ slots,
                                      int32_t slot_stride) {
  ptx::griddep_wait();   // a programmatic dependent of the match kernel
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const float lb = tc_lower_bound(bound, slots, slot_stride, k, q);
  TopK<KT, int32_t> t;
  t.init(true);
  // lists are sorted: walk each from its head while entries can still enter (most lists
  // of a gated batch are empty)
  gather_lists<KT>(part_s, part_i, q, P, k, lb, lane, 32, t);
  warp_emit(t, k, lane, out_s + (int64_t)q * k, out_i + (int64_t)q * k,
            out_hit ? out_hit + q : nullptr, threshold, rank, world, B, true);
}

// Small batches with many partial lists (the small-batch kernel leaves 4-8 per row
// split): one 512-thread block per query instead of one warp, so nq < ~1000 still fills
// the GPU.  Selection by rank, with no serial insert chains (ncu of the insert-based
// version: a 64-query ungated C3 merge took 30 us, one or two dependent-issue warps per
// SM walking 588 lists through register inserts):
//   1. every list head >= lb (the kernels' lower bound) goes to shared memory;
//   2. each head's rank among them (the number of heads ordered before it): the lists
//      are sorted and hold disjoint rows, so a top-k row's list head has rank < k (k heads
//      ordered before it would be k rows ordered before the row), and the row is ordered
//      no later than the k-th head; those <= k lists are "walked";
//   3. entries 0..k-1 of the walked lists that are ordered no later than the k-th head
//      (or >= lb when fewer than k heads exist) are the candidates, <= k * k of them;
//   4. a candidate's rank among the candidates is its output position (keys are distinct
//      rows, so ranks are unique); positions past the candidates are padding.
// The order is (score desc, local index asc) exactly as merge_partials_kernel's
// warp_emit.  More than kMergeMaxHeads heads >= lb (an fp32 call without bounds) falls
// back to per-thread lists on the first 128 threads, merged by warp 0.
constexpr int kMergeBlockThreads = 512;
constexpr int kMergeFallbackThreads = 128;   // KT <= 32: <= 32 KB of fallback staging
constexpr int kMergeMaxHeads = 512;          // rank pass: one head x 512 comparisons per thread

// number of (s[g], i[g]), g < n4 (a multiple of 4, padded with (-inf, -1)), ordered before (v, j)
__device__ __forceinline__ int rank_of(const float* __restrict__ s, const int32_t* __restrict__ i, int n4, float v,
                                       int32_t j) {
  int r = 0;
  for (int g = 0; g < n4; g += 4) {
    const float4 a = *reinterpret_cast<const float4*>(s + g);
    const int4 b = *reinterpret_cast<const int4*>(i + g);
    r += (better(a.x, b.x, v, j) ? 1 : 0) + (better(a.y, b.y, v, j) ? 1 : 0) + (better(a.z, b.z, v, j) ? 1 : 0) +
         (better(a.w, b.w, v, j) ? 1 : 0);
  }
  return r;
}

template <int KT>
__global__ void __launch_bounds__(kMergeBlockThreads)
    merge_partials_block_kernel(const float* __restrict__ part_s, const int32_t* __restrict__ part_i, int32_t nq,
                                int32_t P, int32_t k, float* __restrict__ out_s, int64_t* __restrict__ out_i,
                                uint8_t* __restrict__ out_hit, float threshold, int32_t rank, int32_t world,
                                int64_t B, const uint32_t* __restrict__ bound, const uint32_t* __restrict__ slots,
                                int32_t slot_stride) {
  __shared__ float ss[KT][kMergeFallbackThreads];
  __shared__ int32_t si[KT][kMergeFallbackThreads];
  __shared__ __align__(16) float hs[kMergeMaxHeads + 4];
  __shared__ __align__(16) int32_t hi[kMergeMaxHeads + 4];
  __shared__ int32_t hp[kMergeMaxHeads];
  __shared__ __align__(16) float cs[KT * KT + 4];
  __shared__ __align__(16) int32_t ci[KT * KT + 4];
  __shared__ int32_t walk[KT];
  __shared__ int32_t n_heads, n_cand, kth_i;
  __shared__ float kth_s;
  ptx::griddep_wait();   // a programmatic dependent of the match kernel
  const int q = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31;
  const float lb = tc_lower_bound(bound, slots, slot_stride, k, q);
  float* qs = out_s + (int64_t)q * k;
  int64_t* qi = out_i + (int64_t)q * k;
  if (tid == 0) {
    n_heads = 0;
    n_cand = 0;
  }
  __syncthreads();
  // 1. heads >= lb (up to 4 heads per thread in flight together)
  for (int p0 = tid; p0 < P; p0 += kMergeBlockThreads * 4) {
    float vs[4];
    int32_t vj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + u * kMergeBlockThreads;
      vj[u] = -1;
      vs[u] = -CUDART_INF_F;
      if (p < P) {
        const int64_t base = ((int64_t)q * P + p) * KT;
        vj[u] = part_i[base];
        vs[u] = part_s[base];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (vj[u] < 0 || vs[u] < lb) continue;
      const int h = atomicAdd(&n_heads, 1);
      if (h < kMergeMaxHeads) {
        hs[h] = vs[u];
        hi[h] = vj[u];
        hp[h] = p0 + u * kMergeBlockThreads;
      }
    }
  }
  __syncthreads();
  const int H = n_heads;
  if (H <= kMergeMaxHeads) {
    // 2. ranks of the heads; the walked lists in rank order and the k-th head
    const int H4 = (H + 3) & ~3;
    if (tid < H4 - H) {
      hs[H + tid] = -CUDART_INF_F;
      hi[H + tid] = -1;
    }
    __syncthreads();
    const int W = H < k ? H : k;
    for (int h = tid; h < H; h += kMergeBlockThreads) {
      const float v = hs[h];
      const int32_t j = hi[h];
      const int r = rank_of(hs, hi, H4, v, j);
      if (r < k) walk[r] = hp[h];
      if (r == W - 1) {
        kth_s = H < k ? lb : v;
        kth_i = H < k ? INT32_MAX : j;   // (lb, max): every entry >= lb passes
      }
    }
    __syncthreads();
    // 3. candidates: entries of the walked lists ordered no later than the k-th head
    if (W > 0) {
      const float ts = kth_s;
      const int32_t tj = kth_i;
      for (int e = tid; e < W * k; e += kMergeBlockThreads) {
        const int w = e / k, r = e - w * k;
        const int64_t base = ((int64_t)q * P + walk[w]) * KT + r;
        const int32_t j = part_i[base];
        const float v = part_s[base];
        if (j < 0 || better(ts, tj, v, j)) continue;
        const int c = atomicAdd(&n_cand, 1);   // < W * k <= KT * KT
        cs[c] = v;
        ci[c] = j;
      }
    }
    __syncthreads();
    // 4. output position = rank among the candidates
    const int C = n_cand, C4 = (C + 3) & ~3;
    if (tid < C4 - C) {
      cs[C + tid] = -CUDART_INF_F;
      ci[C + tid] = -1;
    }
    __syncthreads();
    for (int c = tid; c < C; c += kMergeBlockThreads) {
      const float v = cs[c];
      const int32_t j = ci[c];
      const int r = rank_of(cs, ci, C4, v, j);
      if (r < k) {
        qs[r] = v;
        qi[r] = shard_global((int64_t)j, rank, world, B);
        if (r == 0 && out_hit != nullptr) out_hit[q] = v >= threshold ? 1 : 0;
      }
    }
    for (int r = C + tid; r < k; r += kMergeBlockThreads) {
      qs[r] = -CUDART_INF_F;
      qi[r] = -1;
    }
    if (C == 0 && tid == 0 && out_hit != nullptr) out_hit[q] = 0;
    return;
  }
  if (tid >= kMergeFallbackThreads) return;   // no block barriers below
  TopK<KT, int32_t> t;
  t.init(true);
  gather_lists<KT>(part_s, part_i, q, P, k, lb, tid, kMergeFallbackThreads, t);
#pragma unroll
  for (int r = 0; r < KT; ++r) {
    ss[r][tid] = t.s[r];
    si[r][tid] = t.i[r];
  }
  ptx::named_bar_sync(1, kMergeFallbackThreads);
  if (tid >= 32) return;
  TopK<KT, int32_t> m;
  m.init(true);
  for (int w = 0; w < kMergeFallbackThreads / 32; ++w) {
    const int src = w * 32 + lane;
    for (int r = 0; r < k; ++r) {
      const int32_t j = si[r][src];
      const float v = ss[r][src];
      if (j < 0 || !better(v, j, m.kth_s, m.kth_i)) break;
      m.insert(v, j, k);
    }
  }
  warp_emit(m, k, lane, qs, qi, out_hit ? out_hit + q : nullptr, threshold, rank, world, B, true);
}

template <int KT>
__global__ void merge_shards_kernel(const float* __restrict__ in_s, const int64_t* __restrict__ in_i,
                                    int32_t G, int32_t nq, int32_t kin, int32_t k, float* __restrict__ out_s,
                                    int64_t* __restrict__ out_i, uint8_t* __restrict__ out_hit,
                                    float threshold) {
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  TopK<KT, int64_t> t;
  t.init(true);
  for (int g = lane; g < G; g += 32) {
    const int64_t base = ((int64_t)g * nq + q) * kin;
    for (int r = 0; r < kin; ++r) {
      const int64_t j = in_i[base + r];
      const float v = in_s[base + r];
      if (j < 0 || !better(v, j, t.kth_s, t.kth_i)) break;
      t.insert(v, j, k);
    }
  }
  warp_emit(t, k, lane, out_s + (int64_t)q * k, out_i + (int64_t)q * k, out_hit + q, threshold, 0, 1, 1,
            false);
}

inline unsigned blocks_for(int64_t n, int per_block) { return (unsigned)((n + per_block - 1) / per_block); }

}  // namespace

int pick_KT(int k) { return k <= 8 ? 8 : k <= 16 ? 16 : k <= 32 ? 32 : 64; }

cudaError_t launch_append(Pool& p, const void* emb_src, const float* joints_src, int64_t n_src,
                          int64_t first_global, cudaStream_t s) {
  if (n_src <= 0) return cudaSuccess;
  const int wpb = 8;
  const auto& c = p.cfg;
  if (c.dtype == AMS_DTYPE_BF16)
    append_kernel<true><<<blocks_for(n_src, wpb), wpb * 32, 0, s>>>(
        emb_src, joints_src, n_src, first_global, c.dim, c.joint_dim, p.JP, c.rank, c.world, p.B, p.emb,
        p.inv_norm, p.joints);
  else
    append_kernel<false><<<blocks_for(n_src, wpb), wpb * 32, 0, s>>>(
        emb_src, joints_src, n_src, first_global, c.dim, c.joint_dim, p.JP, c.rank, c.world, p.B, p.emb,
        p.inv_norm, p.joints);
  ++p.launches;
  return cudaGetLastError();
}

cudaError_t launch_query_prep(Pool& p, const void* q_src, const float* qj_src, int32_t nq, const int32_t* perm,
                              uint32_t* zero_a, int32_t n_zero_a, uint32_t* zero_b, int32_t n_zero_b,
                              cudaStream_t s) {
  const int wpb = kPrepWarps;
  const auto& c = p.cfg;
  if (c.dtype == AMS_DTYPE_BF16)
    query_prep_kernel<true><<<blocks_for(nq, wpb), wpb * 32, 0, s>>>(
        q_src, qj_src, nq, c.dim, c.joint_dim, p.JP, perm, p.q_stage, p.q_inv, p.q_joints, zero_a, n_zero_a,
        zero_b, n_zero_b);
  else
    query_prep_kernel<false><<<blocks_for(nq, wpb), wpb * 32, 0, s>>>(
        q_src, qj_src, nq, c.dim, c.joint_dim, p.JP, perm, p.q_stage, p.q_inv, p.q_joints, zero_a, n_zero_a,
        zero_b, n_zero_b);
  ++p.launches;
  return cudaGetLastError();
}

cudaError_t launch_query_order(Pool& p, const float* qj_src, int32_t nq, cudaStream_t s) {
  query_order_kernel<<<1, kOrderThreads, 0, s>>>(qj_src, p.cfg.joint_dim, nq, p.q_perm);
  ++p.launches;
  return cudaGetLastError();
}

// fp32 kernels: programmatic dependents of the query prep (launch overlaps its tail)
cudaError_t launch_match_simt(Pool& p, const MatchArgs& a, int32_t S, cudaStream_t s) {
  const int32_t P = S * kSimtThreads;
  const size_t smem = ((size_t)((p.cfg.dim + 3) & ~3) + (size_t)(kSimtThreads / 32) * kSimtChunk) * sizeof(float);
  cudaLaunchAttribute attr[1];
  const cudaLaunchConfig_t cfg = pdl_config(dim3((unsigned)(a.nq * S)), dim3(kSimtThreads), smem, s, attr);
  cudaError_t e = cudaSuccess;
  // the dynamic shared-memory opt-in is set once per pool and size (a host call per match otherwise)
  size_t* opted = p.simt_smem_opt;
#define AMS_SIMT(KT_, SLOT_)                                                                                  \
  if (opted[SLOT_] < smem) {                                                                                  \
    if ((e = cudaFuncSetAttribute(match_simt_f32_kernel<KT_>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                  (int)smem)) != cudaSuccess)                                                 \
      return e;                                                                                               \
    opted[SLOT_] = smem;                                                                                      \
  }                                                                                                           \
  e = cudaLaunchKernelEx(&cfg, match_simt_f32_kernel<KT_>, static_cast<const float*>(p.emb),                 \
                         static_cast<const float*>(p.inv_norm), static_cast<const float*>(p.joints), p.local,  \
                         static_cast<const float*>(p.q_stage), static_cast<const float*>(p.q_inv),             \
                         static_cast<const float*>(p.q_joints), p.cfg.dim, p.JP, S, a.k, a.g2, a.gated, p.part_s, \
                         p.part_i, P)
  switch (a.KT) {
    case 8: AMS_SIMT(8, 0); break;
    case 16: AMS_SIMT(16, 1); break;
    case 32: AMS_SIMT(32, 2); break;
    default: AMS_SIMT(64, 3); break;
  }
#undef AMS_SIMT
  ++p.launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

int f32_tile_lists(int64_t L) { return (int)((L + kTileRows - 1) / kTileRows); }

cudaError_t launch_match_f32_tile(Pool& p, const MatchArgs& a, cudaStream_t s) {
  const int32_t P = f32_tile_lists(p.local);
  cudaLaunchAttribute attr[1];
  const cudaLaunchConfig_t cfg =
      pdl_config(dim3((unsigned)P, (unsigned)((a.nq + kTileQ - 1) / kTileQ)), dim3(kTileThreads), 0, s, attr);
  cudaError_t e = cudaSuccess;
#define AMS_F32T(KT_)                                                                                        \
  e = cudaLaunchKernelEx(&cfg, match_f32_tile_kernel<KT_>, static_cast<const float*>(p.emb),                 \
                         static_cast<const float*>(p.inv_norm), p.local, static_cast<const float*>(p.q_stage), \
                         static_cast<const float*>(p.q_inv), a.nq, p.cfg.dim, a.k, p.part_s, p.part_i, P)
  switch (a.KT) {
    case 8: AMS_F32T(8); break;
    case 16: AMS_F32T(16); break;
    case 32: AMS_F32T(32); break;
    default: AMS_F32T(64); break;
  }
#undef AMS_F32T
  ++p.launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_merge_partials(Pool& p, const MatchArgs& a, int32_t P, float* out_s, int64_t* out_i,
                                  uint8_t* out_hit, bool tc_bounds, cudaStream_t s) {
  const int wpb = 4;
  const auto& c = p.cfg;
  const unsigned g = blocks_for(a.nq, wpb);
  const uint32_t* bnd = tc_bounds ? p.bound : nullptr;
  const uint32_t* sl = (tc_bounds && a.slots) ? p.slots : nullptr;   // filled by launch_match_tc
  // few queries, many lists: a block per query (the warp-per-query grid would leave most
  // SMs idle); KT = 64 keeps the warp kernel (64 KB of staging per block)
  const bool per_block = a.nq < 8 * p.num_sms && P >= 64 && a.KT <= 32;
  // a programmatic dependent of the match kernel: its launch overlaps that kernel's tail
  cudaLaunchAttribute attr[1];
  const cudaLaunchConfig_t cfg = per_block ? pdl_config(dim3((unsigned)a.nq), dim3(kMergeBlockThreads), 0, s, attr)
                                           : pdl_config(dim3(g), dim3(wpb * 32), 0, s, attr);
  cudaError_t e = cudaSuccess;
#define AMS_MERGE(KT_)                                                                                      \
  e = per_block ? cudaLaunchKernelEx(&cfg, merge_partials_block_kernel<KT_ <= 32 ? KT_ : 32>, p.part_s, p.part_i, \
                                     a.nq, P, a.k, out_s, out_i, out_hit, a.threshold, c.rank, c.world, p.B, bnd, \
                                     sl, (int32_t)a.KT)                                                        \
                : cudaLaunchKernelEx(&cfg, merge_partials_kernel<KT_>, p.part_s, p.part_i, a.nq, P, a.k, out_s,  \
                                     out_i, out_hit, a.threshold, c.rank, c.world, p.B, bnd, sl, (int32_t)a.KT)
  switch (a.KT) {
    case 8: AMS_MERGE(8); break;
    case 16: AMS_MERGE(16); break;
    case 32: AMS_MERGE(32); break;
    default: AMS_MERGE(64); break;
  }
#undef AMS_MERGE
  ++p.launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_merge_lists(const MatchArgs& a, int32_t G, int32_t kin, const float* in_s, const int64_t* in_i,
                               float* out_s, int64_t* out_i, uint8_t* out_hit, cudaStream_t s) {
  const int wpb = 4;
  const unsigned g = blocks_for(a.nq, wpb);
#define AMS_MS(KT_)                                                                                   \
  merge_shards_kernel<KT_><<<g, wpb * 32, 0, s>>>(in_s, in_i, G, a.nq, kin, a.k, out_s, out_i, out_hit, \
                                                   a.threshold)
  switch (a.KT) {
    case 8: AMS_MS(8); break;
    case 16: AMS_MS(16); break;
    case 32: AMS_MS(32); break;
    default: AMS_MS(64); break;
  }
#undef AMS_MS
  return cudaGetLastError();
}

cudaError_t launch_merge_shards(Pool& p, const MatchArgs& a, int32_t G, int32_t kin, const float* in_s,
                                const int64_t* in_i, float* out_s, int64_t* out_i, uint8_t* out_hit,
                                cudaStream_t s) {
  ++p.launches;
  return launch_merge_lists(a, G, kin, in_s, in_i, out_s, out_i, out_hit, s);
}

}  // namespace ams
