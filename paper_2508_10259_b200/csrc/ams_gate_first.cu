// ams_gate_first.cu -- gate-first sparse matcher (a variant of the
// dense path, not the north_star contract).
//
// Same function as ams_match: top-k by (score desc, index asc) over the
// rows that pass the canonical fp32 joint gate, cosine scores, hit flags.  When the gate
// is selective (reading R14: ~0-2 eligible rows per query in every config) almost all
// of the dense path's tensor-core work scores ineligible pairs.  This variant evaluates
// the gate for every (query, row) pair first -- reading only the pool's joints (4*JP
// bytes per row instead of 2d) -- and computes dot products for eligible pairs only.
//
//   K1 the gate, one of (by batch; every one appends eligible rows to the query's
//      candidate bucket through an atomic slot, and the bucket order is irrelevant):
//      gate_rows_kernel        <= 16 queries: thread per row, exact gate vs every query;
//      gate_rows_snap_kernel   17..1024 gated queries in joint-0 bins, rows in the
//                              pool's joint-0 snapshot order: warp-uniform query windows;
//      gate_rows_binned_kernel the same for rows outside the snapshot: (row, query)
//                              pairs dealt to lanes;
//      gate_scan_kernel        otherwise: block = QT queries x a row split; pool joint
//                              tiles ([JP][256] fp32, tile-transposed) staged in shared
//                              memory; packed f32x2 4-joint filter per 8 rows, one warp
//                              vote, exact canonical gate for fired rows.
//   K2 score_kernel       warp per query: bf16 dot product per candidate (lanes split d,
//                         fixed butterfly order), s = (acc*inv_q)*inv_e, register top-k;
//                         a bucket that overflowed is recomputed exactly by the warp
//                         scanning every row (rare; exact, on the GPU).
//   then the shard merge path of ams_match (NCCL all-gather + merge) for world > 1.
#include <cuda_bf16.h>
#include <math_constants.h>

#include "ams_internal.cuh"
#include "ams_ptx.cuh"
#include "ams_topk.cuh"

namespace ams {
namespace {

constexpr int kGfThreads = 256;   // threads per gate-scan block (= queries per block at QT = 256)
constexpr int kGfTile = kRowAlign; // 256 rows per staged joint tile

// The rows a scan visits: a contiguous range of a tile-transposed joint array, either
// the pool itself (ids == nullptr, plain mode: rows [begin, end)) or the joint-0 index
// snapshot (ids = snapshot position -> local row; bin_off != nullptr: each block derives
// its range from its queries' joint-0 interval).
struct GfRows {
  const float* jt;         // [tiles][JP][256]
  const int32_t* ids;      // nullptr: row = local row
  int64_t begin, end;      // plain mode range
  const int32_t* bin_off;  // snapshot mode: [kSnapBins + 1]
  const float* meta;       // snapshot mode: {lo, scale} of the bins
};

// linear bin of v among kSnapBins bins (lo, scale); NaN and out-of-range values clamp.
// Monotone in v, identical in the build and in the lookup.
__device__ __forceinline__ int snap_bin(float v, float lo, float scale) {
  const float f = (v - lo) * scale;
  return (f >= 0.0f && f < (float)kSnapBins) ? (int)f : (f >= 0.0f ? kSnapBins - 1 : 0);
}

// QT queries per block (32..256): warp w takes query slot w % (QT/32) and, when QT < 256,
// row part w / (QT/32) of every staged tile, so a small batch keeps all 8 warps busy on
// its few queries instead of running 256-thread blocks of mostly inactive warps.
template <int JP, int QT>
__global__ void __launch_bounds__(kGfThreads)
    gate_scan_kernel(const GfRows rows, const float* __restrict__ q_joints, int32_t nq, int32_t S, float g2,
                     int32_t cap, uint32_t* __restrict__ cnt, int32_t* __restrict__ cand, int32_t sorted) {
  __shared__ __align__(16) float js[2][JP * kGfTile];
  __shared__ __align__(16) float pn[kGfTile];       // per row: sum of squares of the first 4 joints
  __shared__ unsigned int pmax_bits;
  __shared__ float blk_lo[kGfThreads / 32], blk_hi[kGfThreads / 32];
  constexpr int kSlots = QT / 32, kParts = kGfThreads / QT;   // query slots x row parts = 8 warps
  constexpr int kC8 = kGfTile / 8 / kParts;                    // 8-row groups per row part
  static_assert(kC8 % 4 == 0, "row parts must hold whole 32-row groups");
  ptx::griddep_wait();   // a programmatic dependent of the query prep (joints, zeroed counts)
  const float* __restrict__ pool_joints = rows.jt;
  const int qg = blockIdx.x, sp = blockIdx.y;
  const int q = qg * QT + ((int)(threadIdx.x >> 5) % kSlots) * 32 + (int)(threadIdx.x & 31);
  const int c8_lo = ((int)(threadIdx.x >> 5) / kSlots) * kC8;
  const bool active = q < nq;
  float qj[JP];
#pragma unroll
  for (int t = 0; t < JP; ++t) qj[t] = active ? q_joints[(int64_t)q * JP + t] : 0.0f;
  uint64_t QQ[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) QQ[t] = ptx::pack2(qj[t], qj[t]);
  float rq = 0.0f;
#pragma unroll
  for (int t = 0; t < 4; ++t) rq = fmaf(qj[t], qj[t], rq);
  const uint64_t M2 = ptx::pack2(-2.0f, -2.0f);
  // joint-0 / joint-1 intervals of the warp's active queries (see ams_match_tc.cu epi_chunk_sorted)
  float wlo = active ? qj[0] : CUDART_INF_F, whi = active ? qj[0] : -CUDART_INF_F;
  float wlo1 = active ? qj[1] : CUDART_INF_F, whi1 = active ? qj[1] : -CUDART_INF_F;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    wlo = fminf(wlo, __shfl_xor_sync(0xffffffffu, wlo, o));
    whi = fmaxf(whi, __shfl_xor_sync(0xffffffffu, whi, o));
    wlo1 = fminf(wlo1, __shfl_xor_sync(0xffffffffu, wlo1, o));
    whi1 = fmaxf(whi1, __shfl_xor_sync(0xffffffffu, whi1, o));
  }
  const int lane = threadIdx.x & 31;
  int64_t R0 = rows.begin, R1 = rows.end;
  if (rows.bin_off != nullptr) {
    // snapshot: rows whose joint 0 lies within gamma of the block's joint-0 interval.  A
    // row can pass only if RN(RN(r0 - p0)^2) <= g2, i.e. |r0 - p0| <= sqrt(g2)(1 + 2^-23);
    // gp rounds that up, and one extra bin on each side absorbs the rounding of the bin
    // arithmetic, so every eligible row is inside [R0, R1).
    if (lane == 0) {
      blk_lo[threadIdx.x >> 5] = wlo;
      blk_hi[threadIdx.x >> 5] = whi;
    }
    __syncthreads();
    float blo = blk_lo[0], bhi = blk_hi[0];
    for (int w = 1; w < kGfThreads / 32; ++w) {
      blo = fminf(blo, blk_lo[w]);
      bhi = fmaxf(bhi, blk_hi[w]);
    }
    if (!(blo <= bhi)) {
      R0 = R1 = 0;   // no active query in this block
    } else {
      const float lo = rows.meta[0], scale = rows.meta[1];
      const float gp = __fmul_ru(__fsqrt_ru(g2), 1.00000095367431640625f);   // (1 + 2^-20)
      const int ba = max(0, snap_bin(__fsub_rd(blo, gp), lo, scale) - 1);
      const int bb = min(kSnapBins - 1, snap_bin(__fadd_ru(bhi, gp), lo, scale) + 1);
      R0 = rows.bin_off[ba];
      R1 = rows.bin_off[bb + 1];
    }
  }
  const int64_t T0 = R0 / kGfTile, n_pt = R1 > R0 ? (R1 + kGfTile - 1) / kGfTile - T0 : 0;
  const int64_t t_lo = T0 + n_pt * sp / S, t_hi = T0 + n_pt * (sp + 1) / S;
  auto stage = [&](int64_t t, int buf) {   // cp.async (LDGSTS): does not block the thread
    const float4* src = reinterpret_cast<const float4*>(pool_joints + t * kGfTile * JP);
    float4* dst = reinterpret_cast<float4*>(js[buf]);
    for (int i = threadIdx.x; i < JP * kGfTile / 4; i += kGfThreads)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(dst + i)), "l"(src + i)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (t_lo < t_hi) stage(t_lo, 0);
  for (int64_t t = t_lo; t < t_hi; ++t) {
    const int buf = (int)((t - t_lo) & 1);
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (threadIdx.x == 0) pmax_bits = 0u;
    __syncthreads();   // tile t landed for every thread; everyone is done with tile t-1
    if (t + 1 < t_hi) stage(t + 1, buf ^ 1);   // prefetch the next tile into the other buffer
    const float* jsm = js[buf];
    {  // per-row partial norms (one row per thread; any fp32 order -- covered by eps)
      float v = 0.0f;
#pragma unroll
      for (int u = 0; u < 4; ++u) v = fmaf(jsm[u * kGfTile + threadIdx.x], jsm[u * kGfTile + threadIdx.x], v);
      pn[threadIdx.x] = v;
      const unsigned int wmax = __reduce_max_sync(0xffffffffu, __float_as_uint(v));   // v >= 0: int order = float order
      if ((threadIdx.x & 31) == 0) atomicMax(&pmax_bits, wmax);
    }
    __syncthreads();
    // Superset filter in expanded form over the first 4 joints: v = P_j - 2 r.p_j <= tq,
    // tq = g2 - R + eps.  |(v' + R') - partial canonical sum| <= ~24 u (g2 + R + Pmax),
    // u = 2^-24; eps = 2^-18 (g2 + R + Pmax) covers it with margin.  Rows that pass get the
    // exact canonical gate below, so the result is exact.
    const float tq = active ? (g2 - rq) + 3.814697265625e-06f * (g2 + rq + __uint_as_float(pmax_bits))
                            : -CUDART_INF_F;
    const int64_t row0 = t * kGfTile;
    const int cmin = (int)max((int64_t)0, R0 - row0);                 // rows [cmin, nvalid) of the tile
    const int nvalid = (int)min((int64_t)kGfTile, R1 - row0);
    auto emit = [&](int c) {   // eligible row c of the tile for this lane's query
      const uint32_t slot = atomicAdd(&cnt[q], 1u);
      if (slot < (uint32_t)cap)
        cand[(int64_t)q * cap + slot] = rows.ids != nullptr ? rows.ids[row0 + c] : (int32_t)(row0 + c);
    };
    auto exact = [&](int c) {   // canonical gate of row c for this lane's query
      float ds = 0.0f;
#pragma unroll
      for (int u = 0; u < JP; ++u) {
        const float df = __fsub_rn(qj[u], jsm[u * kGfTile + c]);
        ds = __fmaf_rn(df, df, ds);
      }
      if (active && c >= cmin && c < nvalid && ds <= g2) emit(c);
    };
#pragma unroll 1
    for (int c8 = c8_lo; c8 < c8_lo + kC8; ++c8) {
      if (sorted && (c8 & 3) == 0) {
        // warp-level two-joint test of the next 32 rows (ams_match_tc.cu
        // epi_chunk_sorted): ineligible for every lane when it fails
        const float p0 = jsm[8 * c8 + lane], p1 = jsm[kGfTile + 8 * c8 + lane];
        const float d0 = p0 < wlo ? __fsub_rn(wlo, p0) : (p0 > whi ? __fsub_rn(whi, p0) : 0.0f);
        const float d1 = p1 < wlo1 ? __fsub_rn(wlo1, p1) : (p1 > whi1 ? __fsub_rn(whi1, p1) : 0.0f);
        uint32_t m = __ballot_sync(0xffffffffu, __fmaf_rn(d1, d1, __fmul_rn(d0, d0)) <= g2);
        if (__popc(m) <= 10) {
          while (m != 0u) {
            const int c = 8 * c8 + __ffs(m) - 1;
            m &= m - 1u;
            // canonical gate with a warp-uniform early exit every 4 joints (partial sums
            // of squares only grow)
            float ds = 0.0f;
            bool ok = active && c >= cmin && c < nvalid;
#pragma unroll
            for (int g4 = 0; g4 < JP / 4; ++g4) {
              if (!__any_sync(0xffffffffu, ok)) break;
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float df = __fsub_rn(qj[4 * g4 + u], jsm[(4 * g4 + u) * kGfTile + c]);
                ds = __fmaf_rn(df, df, ds);
              }
              ok = ok && (ds <= g2);
            }
            if (ok) emit(c);
          }
          c8 += 3;
          continue;
        }
      }
      float mn = CUDART_INF_F;
#pragma unroll
      for (int c4 = 2 * c8; c4 < 2 * c8 + 2; ++c4) {
        const float4 p0 = *reinterpret_cast<const float4*>(jsm + 4 * c4);
        const float4 pv = *reinterpret_cast<const float4*>(pn + 4 * c4);
        uint64_t a = ptx::mul2(QQ[0], ptx::pack2(p0.x, p0.y));
        uint64_t b = ptx::mul2(QQ[0], ptx::pack2(p0.z, p0.w));
#pragma unroll
        for (int t4 = 1; t4 < 4; ++t4) {
          const float4 p = *reinterpret_cast<const float4*>(jsm + t4 * kGfTile + 4 * c4);
          a = ptx::fma2(QQ[t4], ptx::pack2(p.x, p.y), a);
          b = ptx::fma2(QQ[t4], ptx::pack2(p.z, p.w), b);
        }
        a = ptx::fma2(a, M2, ptx::pack2(pv.x, pv.y));
        b = ptx::fma2(b, M2, ptx::pack2(pv.z, pv.w));
        mn = fminf(mn, fminf(fminf(ptx::lo2(a), ptx::hi2(a)), fminf(ptx::lo2(b), ptx::hi2(b))));
      }
      if (!__any_sync(0xffffffffu, mn <= tq)) continue;
      // exact canonical gate for the 8 rows of this group
#pragma unroll 1
      for (int c = 8 * c8; c < 8 * c8 + 8; ++c) exact(c);
    }
  }
  ptx::griddep_launch_dependents();
}

// Tiny batches (nq <= kGfRowsMaxQ) on the plain row range: thread per row, the exact
// canonical gate of the row against every query, no staging and no block barriers, so
// the scan streams the pool's joints (4 JP bytes per row) at HBM speed instead of paying
// the warp-per-32-queries kernel's per-tile overhead for one or two live lanes (C5 pool,
// 1 query: 64 us there).  Eligible rows go to the query's bucket as in gate_scan_kernel
// (bucket order is irrelevant: the score kernel orders by (score, index)).
constexpr int kGfRowsThreads = 256;   // (kGfRowsMaxQ: ams_internal.cuh)

template <int JP>
__global__ void __launch_bounds__(kGfRowsThreads)
    gate_rows_kernel(const float* __restrict__ pool_joints, int64_t L, const float* __restrict__ q_joints,
                     int32_t nq, float g2, int32_t cap, uint32_t* __restrict__ cnt, int32_t* __restrict__ cand) {
  __shared__ float qs[kGfRowsMaxQ * JP];
  ptx::griddep_wait();   // a programmatic dependent of the query prep
  for (int i = threadIdx.x; i < nq * JP; i += kGfRowsThreads) qs[i] = q_joints[i];
  __syncthreads();
  constexpr int kU = 4;   // rows per thread in flight
  const int64_t stride = (int64_t)gridDim.x * kGfRowsThreads;
  for (int64_t j0 = (int64_t)blockIdx.x * kGfRowsThreads + threadIdx.x; j0 < L; j0 += kU * stride) {
    float pj[kU][JP];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t j = j0 + u * stride;
#pragma unroll
      for (int t = 0; t < JP; ++t) pj[u][t] = j < L ? __ldcs(pool_joints + joint_offset(j, t, JP)) : 0.0f;
    }
    for (int qi = 0; qi < nq; ++qi) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        float ds = 0.0f;
#pragma unroll
        for (int t = 0; t < JP; ++t) {
          const float df = __fsub_rn(qs[qi * JP + t], pj[u][t]);
          ds = __fmaf_rn(df, df, ds);
        }
        if (ds <= g2 && j0 + u * stride < L) {   // (g2 may be +inf: the row bound is explicit)
          const uint32_t slot = atomicAdd(&cnt[qi], 1u);
          if (slot < (uint32_t)cap) cand[(int64_t)qi * cap + slot] = (int32_t)(j0 + u * stride);
        }
      }
    }
  }
  ptx::griddep_launch_dependents();
}

// ------------------------------------------------------------ mid-size batches (17..1024)
// The queries are staged in kQBins linear joint-0 bins (query_order_j0_kernel); a pool
// row can pass the canonical gate only for queries whose joint 0 is within gamma of its
// own (the canonical partial sums only grow: RN(RN(q0 - r0)^2) > g2 fails the gate), so
// gate_rows_binned_kernel visits, per row, only the queries of the bins overlapping
// [r0 - gp, r0 + gp] (gp = sqrt(g2) rounded up, widened by 2^-20, plus one bin on each
// side for the rounding of the bin arithmetic -- the argument of the pool-side joint-0
// index) and runs the exact gate with an early exit once a partial sum exceeds g2.  Per
// row that is ~nq * 2 gamma / span(joint 0) queries instead of nq, so the scan stays
// bound by reading the joints (C5 pool, 256 queries: 309 us in the warp kernel, whose
// ALU cost is per (row, query) pair).
__device__ __forceinline__ int qbin(float v, float lo, float scale) {
  const float f = (v - lo) * scale;
  return (f >= 0.0f && f < (float)kQBins) ? (int)f : (f >= 0.0f ? kQBins - 1 : 0);
}

constexpr int kQOrderThreads = 256;

__global__ void __launch_bounds__(kQOrderThreads)
    query_order_j0_kernel(const float* __restrict__ jsrc, int32_t J, int32_t nq, int32_t* __restrict__ perm,
                          int32_t* __restrict__ qbins) {
  __shared__ uint32_t hist[kQBins];
  __shared__ float red_lo[kQOrderThreads / 32], red_hi[kQOrderThreads / 32];
  __shared__ uint32_t wsum[kQOrderThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  float l = CUDART_INF_F, h = -CUDART_INF_F;
  for (int q = tid; q < nq; q += kQOrderThreads) {
    const float v = jsrc[(int64_t)q * J];
    if (v == v) {
      l = fminf(l, v);
      h = fmaxf(h, v);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l = fminf(l, __shfl_xor_sync(0xffffffffu, l, o));
    h = fmaxf(h, __shfl_xor_sync(0xffffffffu, h, o));
  }
  if (lane == 0) {
    red_lo[w] = l;
    red_hi[w] = h;
  }
  for (int b = tid; b < kQBins; b += kQOrderThreads) hist[b] = 0u;
  __syncthreads();
  l = red_lo[0];
  h = red_hi[0];
  for (int i = 1; i < kQOrderThreads / 32; ++i) {
    l = fminf(l, red_lo[i]);
    h = fmaxf(h, red_hi[i]);
  }
  const float span = h - l;
  const float lo = l < CUDART_INF_F ? l : 0.0f;
  const float scale = (span > 1e-30f && span < CUDART_INF_F) ? (float)kQBins / span : 0.0f;
  for (int q = tid; q < nq; q += kQOrderThreads) atomicAdd(&hist[qbin(jsrc[(int64_t)q * J], lo, scale)], 1u);
  __syncthreads();
  // exclusive scan: thread t owns bins [4t, 4t + 4)
  constexpr int per = kQBins / kQOrderThreads;
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
    qbins[tid * per + i] = (int32_t)base;
    hist[tid * per + i] = base;
    base += v[i];
  }
  if (tid == 0) {
    qbins[kQBins] = nq;
    qbins[kQBins + 1] = __float_as_int(lo);
    qbins[kQBins + 2] = __float_as_int(scale);
  }
  __syncthreads();
  for (int q = tid; q < nq; q += kQOrderThreads) {
    const uint32_t pos = atomicAdd(&hist[qbin(jsrc[(int64_t)q * J], lo, scale)], 1u);
    perm[pos] = q;   // order within a bin is irrelevant: a row visits whole bins
  }
}

// Per warp, 32 consecutive rows per step (coalesced joint loads; the rows' joints go to
// shared memory); each lane's row contributes the queries of its joint-0 window, and the
// warp's (row, query) pairs are then dealt 32 at a time to the lanes (owner row by a
// 5-step search over the lanes' prefix sums), so the gate arithmetic runs on full warps
// instead of one divergent per-lane loop (ncu of that version: 26 % lane efficiency).
template <int JP>
__global__ void __launch_bounds__(kGfRowsThreads)
    gate_rows_binned_kernel(const float* __restrict__ pool_joints, int64_t begin, int64_t L,
                            const float* __restrict__ q_joints, int32_t nq, float g2, int32_t cap,
                            uint32_t* __restrict__ cnt, int32_t* __restrict__ cand, const int32_t* __restrict__ qbins) {
  constexpr int QS = JP + 1;   // padded strides (conflict-free for distinct rows / queries)
  extern __shared__ __align__(16) float qs[];                        // [nq][QS] staged (binned) order
  int32_t* off = reinterpret_cast<int32_t*>(qs + (size_t)nq * QS);   // [kQBins + 1]
  __shared__ float rows_s[kGfRowsThreads / 32][32 * QS];
  __shared__ int32_t pre_s[kGfRowsThreads / 32][32], qa_s[kGfRowsThreads / 32][32];
  ptx::griddep_wait();   // a programmatic dependent of the query prep
  for (int i = threadIdx.x; i < nq * JP; i += kGfRowsThreads) qs[(i / JP) * QS + i % JP] = q_joints[i];
  for (int i = threadIdx.x; i <= kQBins; i += kGfRowsThreads) off[i] = qbins[i];
  const float lo = __int_as_float(qbins[kQBins + 1]), scale = __int_as_float(qbins[kQBins + 2]);
  const float gp = __fmul_ru(__fsqrt_ru(g2), 1.00000095367431640625f);   // (1 + 2^-20)
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* rs = rows_s[wib];
  int32_t* pre = pre_s[wib];
  int32_t* qa_w = qa_s[wib];
  const int64_t nwarps = (int64_t)gridDim.x * (kGfRowsThreads / 32);
  for (int64_t base = begin + ((int64_t)blockIdx.x * (kGfRowsThreads / 32) + wib) * 32; base < L;
       base += nwarps * 32) {
    const int64_t j = base + lane;
    int c = 0, qa = 0;
    if (j < L) {
#pragma unroll
      for (int t = 0; t < JP; ++t) rs[lane * QS + t] = __ldcs(pool_joints + joint_offset(j, t, JP));
      const float r0 = rs[lane * QS];
      const int ba = max(0, qbin(__fsub_rd(r0, gp), lo, scale) - 1);
      const int bb = min(kQBins - 1, qbin(__fadd_ru(r0, gp), lo, scale) + 1);
      qa = off[ba];
      c = off[bb + 1] - qa;
    }
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    pre[lane] = incl - c;
    qa_w[lane] = qa;
    __syncwarp();
    for (int p = lane; p < total; p += 32) {
      int r = 0;   // the last lane whose pair range starts at or before p
#pragma unroll
      for (int st = 16; st > 0; st >>= 1)
        if (pre[r + st] <= p) r += st;
      const int qi = qa_w[r] + (p - pre[r]);
      const float* rj = rs + r * QS;
      const float* qj = qs + qi * QS;
      // the canonical gate (joint order, fsub then fmaf); partial sums only grow, so
      // most pairs stop after joint 1
      float df = __fsub_rn(qj[0], rj[0]);
      float ds = __fmaf_rn(df, df, 0.0f);
      if (JP > 1) {
        df = __fsub_rn(qj[1], rj[1]);
        ds = __fmaf_rn(df, df, ds);
      }
      if (!(ds <= g2)) continue;
#pragma unroll
      for (int t = 2; t < JP; ++t) {
        df = __fsub_rn(qj[t], rj[t]);
        ds = __fmaf_rn(df, df, ds);
      }
      if (ds <= g2) {
        const uint32_t slot = atomicAdd(&cnt[qi], 1u);
        if (slot < (uint32_t)cap) cand[(int64_t)qi * cap + slot] = (int32_t)(base + r);
      }
    }
    __syncwarp();
  }
  ptx::griddep_launch_dependents();
}

// Rows in joint-0 order (the pool-side snapshot index, positions [0, snap_L)): the 32 rows
// of a warp span a tiny joint-0 interval, so their windows nearly coincide and the warp
// walks the union window with a warp-uniform loop -- every lane tests its own row against
// the same query (a broadcast shared-memory read) -- instead of dealing pairs.
template <int JP>
__global__ void __launch_bounds__(kGfRowsThreads)
    gate_rows_snap_kernel(const float* __restrict__ snap_j, const int32_t* __restrict__ snap_id, int64_t L,
                          const float* __restrict__ q_joints, int32_t nq, float g2, int32_t cap,
                          uint32_t* __restrict__ cnt, int32_t* __restrict__ cand, const int32_t* __restrict__ qbins) {
  extern __shared__ __align__(16) float qs[];                              // [nq][JP] staged (binned) order
  int32_t* off = reinterpret_cast<int32_t*>(qs + (size_t)nq * (JP + 1));   // [kQBins + 1]
  ptx::griddep_wait();   // a programmatic dependent of the query prep
  for (int i = threadIdx.x; i < nq * JP; i += kGfRowsThreads) qs[i] = q_joints[i];
  for (int i = threadIdx.x; i <= kQBins; i += kGfRowsThreads) off[i] = qbins[i];
  const float lo = __int_as_float(qbins[kQBins + 1]), scale = __int_as_float(qbins[kQBins + 2]);
  const float gp = __fmul_ru(__fsqrt_ru(g2), 1.00000095367431640625f);   // (1 + 2^-20)
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * (kGfRowsThreads / 32);
  // the next group's joints are loaded before the current group's windows are walked
  // (software pipelining: ncu showed the warps waiting on these loads)
  const int64_t first = ((int64_t)blockIdx.x * (kGfRowsThreads / 32) + wib) * 32;
  float pj_next[JP];
#pragma unroll
  for (int t = 0; t < JP; ++t)
    pj_next[t] = first + lane < L ? __ldcs(snap_j + joint_offset(first + lane, t, JP)) : 0.0f;
  for (int64_t base = first; base < L; base += nwarps * 32) {
    const int64_t pos = base + lane;
    const bool valid = pos < L;
    float pj[JP];
#pragma unroll
    for (int t = 0; t < JP; ++t) pj[t] = pj_next[t];
    const int64_t npos = pos + nwarps * 32;
#pragma unroll
    for (int t = 0; t < JP; ++t) pj_next[t] = npos < L ? __ldcs(snap_j + joint_offset(npos, t, JP)) : 0.0f;
    // the union of the lanes' windows (NaN joints pass no gate: fminf / fmaxf drop them)
    float wmin = valid ? pj[0] : CUDART_INF_F, wmax = valid ? pj[0] : -CUDART_INF_F;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      wmin = fminf(wmin, __shfl_xor_sync(0xffffffffu, wmin, o));
      wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    }
    if (!(wmin <= wmax)) continue;
    const int ba = max(0, qbin(__fsub_rd(wmin, gp), lo, scale) - 1);
    const int bb = min(kQBins - 1, qbin(__fadd_ru(wmax, gp), lo, scale) + 1);
    const int qa = off[ba], qb = off[bb + 1];
    for (int qi = qa; qi < qb; ++qi) {
      const float* qj = qs + qi * JP;
      // the canonical gate (joint order, fsub then fmaf); partial sums only grow
      float df = __fsub_rn(qj[0], pj[0]);
      float ds = __fmaf_rn(df, df, 0.0f);
      if (JP > 1) {
        df = __fsub_rn(qj[1], pj[1]);
        ds = __fmaf_rn(df, df, ds);
      }
      if (!(ds <= g2 && valid)) continue;
#pragma unroll
      for (int t = 2; t < JP; ++t) {
        df = __fsub_rn(qj[t], pj[t]);
        ds = __fmaf_rn(df, df, ds);
      }
      if (ds <= g2) {
        const uint32_t slot = atomicAdd(&cnt[qi], 1u);
        if (slot < (uint32_t)cap) cand[(int64_t)qi * cap + slot] = snap_id[pos];
      }
    }
  }
  ptx::griddep_launch_dependents();
}

__device__ __forceinline__ float bf16_dot_lane(const uint4* __restrict__ a, const uint4* __restrict__ b, int n16,
                                               int lane) {
  // lanes take 16-byte pieces lane, lane+32, ...; fp32 accumulation in a fixed order.
  // Pieces are loaded 8 at a time before their FMAs (one round trip per 8 instead of per
  // piece: a d = 4096 row is 16 pieces per lane); the FMA order is unchanged.
  float acc = 0.0f;
  constexpr int kB = 8;
  for (int i0 = lane; i0 < n16; i0 += 32 * kB) {
    uint4 x[kB], y[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int i = i0 + 32 * u;
      x[u] = i < n16 ? __ldg(a + i) : make_uint4(0u, 0u, 0u, 0u);
      y[u] = i < n16 ? __ldg(b + i) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      if (i0 + 32 * u >= n16) break;
      const uint32_t xs[4] = {x[u].x, x[u].y, x[u].z, x[u].w}, ys[4] = {y[u].x, y[u].y, y[u].z, y[u].w};
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        acc = __fmaf_rn(__uint_as_float(xs[v] << 16), __uint_as_float(ys[v] << 16), acc);
        acc = __fmaf_rn(__uint_as_float(xs[v] & 0xFFFF0000u), __uint_as_float(ys[v] & 0xFFFF0000u), acc);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

template <int KT, int JP>
__global__ void score_kernel(const uint16_t* __restrict__ emb, const float* __restrict__ inv_e,
                             const float* __restrict__ pool_joints, int64_t L, const uint16_t* __restrict__ q,
                             const float* __restrict__ inv_q, const float* __restrict__ q_joints, int32_t d,
                             int32_t nq, int32_t k, float g2, int32_t cap, const uint32_t* __restrict__ cnt,
                             const int32_t* __restrict__ cand, float* __restrict__ out_s, int64_t* __restrict__ out_i,
                             uint8_t* __restrict__ out_hit, float threshold, int32_t rank, int32_t world,
                             int64_t B, const int32_t* __restrict__ perm) {
  ptx::griddep_wait();   // a programmatic dependent of the gate scan (buckets complete)
  const int lane = threadIdx.x & 31;
  const int qi = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (qi >= nq) return;
  const int64_t qo = perm != nullptr ? (int64_t)perm[qi] : (int64_t)qi;   // caller's query index
  const int n16 = d / 8;
  const uint4* qv = reinterpret_cast<const uint4*>(q + (int64_t)qi * d);
  const float iq = inv_q[qi];
  TopK<KT, int32_t> top;
  top.init(true);
  const uint32_t n = cnt[qi];
  if (n <= (uint32_t)cap) {
    for (uint32_t c = 0; c < n; ++c) {
      const int32_t j = cand[(int64_t)qi * cap + c];
      const float acc = bf16_dot_lane(qv, reinterpret_cast<const uint4*>(emb + (int64_t)j * d), n16, lane);
      const float s = __fmul_rn(__fmul_rn(acc, iq), inv_e[j]);
      if (lane == 0 && better(s, j, top.kth_s, top.kth_i)) top.insert(s, j, k);
    }
  } else {
    // bucket overflow: exact exhaustive scan of this query (lane per row, increasing)
    float r[JP];
#pragma unroll
    for (int t = 0; t < JP; ++t) r[t] = q_joints[(int64_t)qi * JP + t];
    for (int64_t j = lane; j < L; j += 32) {
      float ds = 0.0f;
#pragma unroll
      for (int t = 0; t < JP; ++t) {
        const float df = __fsub_rn(r[t], pool_joints[joint_offset(j, t, JP)]);
        ds = __fmaf_rn(df, df, ds);
      }
      if (!(ds <= g2)) continue;
      const uint32_t* e = reinterpret_cast<const uint32_t*>(emb + j * d);
      const uint32_t* qq = reinterpret_cast<const uint32_t*>(q + (int64_t)qi * d);
      // same per-lane order as bf16_dot_lane would give is not required: any fp32 order
      float acc = 0.0f;
      for (int w = 0; w < d / 2; ++w) {
        acc = __fmaf_rn(__uint_as_float(qq[w] << 16), __uint_as_float(e[w] << 16), acc);
        acc = __fmaf_rn(__uint_as_float(qq[w] & 0xFFFF0000u), __uint_as_float(e[w] & 0xFFFF0000u), acc);
      }
      const float s = __fmul_rn(__fmul_rn(acc, iq), inv_e[j]);
      if (s > top.kth_s) top.insert_monotone(s, (int32_t)j, k);
    }
  }
  if (n <= (uint32_t)cap) {
    // bucket path: lane 0's list is the whole (sorted) result -- write it directly
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < KT; ++r) {
        if (r >= k) break;
        const bool v = top.i[r] >= 0;
        out_s[qo * k + r] = v ? top.s[r] : -CUDART_INF_F;
        out_i[qo * k + r] = v ? shard_global((int64_t)top.i[r], rank, world, B) : -1;
      }
      if (out_hit != nullptr) out_hit[qo] = (top.i[0] >= 0 && top.s[0] >= threshold) ? 1 : 0;
    }
    return;
  }
  // overflow path: k rounds of a butterfly arg-max over the lanes' lists
  float s0 = -CUDART_INF_F;
  int64_t i0 = -1;
  for (int r = 0; r < k; ++r) {
    float bs = top.s[0];
    int32_t bi = top.i[0];
    int bl = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float os = __shfl_xor_sync(0xffffffffu, bs, o);
      const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (better(os, oi, bs, bi) || (!better(bs, bi, os, oi) && ol < bl)) {
        bs = os;
        bi = oi;
        bl = ol;
      }
    }
    const int64_t gi = bi >= 0 ? shard_global((int64_t)bi, rank, world, B) : -1;
    if (lane == 0) {
      out_s[qo * k + r] = bi >= 0 ? bs : -CUDART_INF_F;
      out_i[qo * k + r] = gi;
    }
    if (r == 0) {
      s0 = bs;
      i0 = gi;
    }
    if (lane == bl) top.pop_front();
  }
  if (out_hit != nullptr && lane == 0) out_hit[qo] = (i0 >= 0 && s0 >= threshold) ? 1 : 0;
}

// ------------------------------------------------------------------ joint-0 index build
// A bucket sort of the local rows [0, L) by joint 0 (any order within a bin is fine: a
// scan covers whole bins).  aux layout: [0, kSnapBins) histogram then cursor,
// [kSnapBins, kSnapBins + 2) {min, max} of joint 0 as ordered u32, then {lo, scale} as
// floats at [kSnapBins + 2, kSnapBins + 4).
constexpr int kSnapMinRows = 65536;   // smaller pools: the plain scan is cheap enough

__global__ void snap_minmax_kernel(const float* __restrict__ joints, int64_t L, int32_t JP, uint32_t* __restrict__ mm) {
  uint32_t lo = 0xFFFFFFFFu, hi = 0u;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < L; l += (int64_t)gridDim.x * blockDim.x) {
    const float v = joints[joint_offset(l, 0, JP)];
    if (v == v) {
      lo = min(lo, ptx::f2ord(v));
      hi = max(hi, ptx::f2ord(v));
    }
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], lo);
    atomicMax(&mm[1], hi);
  }
}

__device__ __forceinline__ void snap_params(const uint32_t* mm, float& lo, float& scale) {
  lo = mm[0] == 0xFFFFFFFFu ? 0.0f : ptx::ord2f(mm[0]);
  const float hi = mm[1] == 0u ? 0.0f : ptx::ord2f(mm[1]);
  const float span = hi - lo;
  scale = (span > 1e-30f && span < CUDART_INF_F) ? (float)kSnapBins / span : 0.0f;
}

__global__ void snap_hist_kernel(const float* __restrict__ joints, int64_t L, int32_t JP, uint32_t* __restrict__ aux) {
  float lo, scale;
  snap_params(aux + kSnapBins, lo, scale);
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < L; l += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&aux[snap_bin(joints[joint_offset(l, 0, JP)], lo, scale)], 1u);
}

// one block of 1024 threads: exclusive scan of the histogram into bin_off (and the cursor)
__global__ void __launch_bounds__(1024) snap_scan_kernel(uint32_t* __restrict__ aux, int32_t* __restrict__ bin_off) {
  constexpr int per = kSnapBins / 1024;
  __shared__ uint32_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t run = 0;
  for (int i = 0; i < per; ++i) run += aux[tid * per + i];
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
  for (int i = 0; i < per; ++i) {
    const uint32_t c = aux[tid * per + i];
    bin_off[tid * per + i] = (int32_t)base;
    aux[tid * per + i] = base;   // cursor
    base += c;
  }
  if (tid == 1023) bin_off[kSnapBins] = (int32_t)base;
  if (tid == 0) {
    float lo, scale;
    snap_params(aux + kSnapBins, lo, scale);
    reinterpret_cast<float*>(aux + kSnapBins + 2)[0] = lo;
    reinterpret_cast<float*>(aux + kSnapBins + 2)[1] = scale;
  }
}

__global__ void snap_scatter_kernel(const float* __restrict__ joints, int64_t L, int32_t JP,
                                    uint32_t* __restrict__ aux, float* __restrict__ snap_j,
                                    int32_t* __restrict__ snap_id) {
  float lo, scale;
  snap_params(aux + kSnapBins, lo, scale);
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < L; l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = atomicAdd(&aux[snap_bin(joints[joint_offset(l, 0, JP)], lo, scale)], 1u);
    snap_id[pos] = (int32_t)l;
    for (int t = 0; t < JP; ++t) snap_j[joint_offset(pos, t, JP)] = joints[joint_offset(l, t, JP)];
  }
}

// (Re)build the index over the current local rows when it is missing or its unsorted
// tail has grown past max(64 K, L / 32) rows.  Lazily allocated on first use.
cudaError_t snap_refresh(Pool& p, cudaStream_t s) {
  const int64_t L = p.local;
  if (p.snap_L > 0 && L - p.snap_L <= std::max<int64_t>(65536, L / 32)) return cudaSuccess;
  cudaError_t e;
  if (p.snap_j == nullptr) {
    if ((e = cudaMalloc((void**)&p.snap_j, (size_t)p.cap_pad * p.JP * 4)) != cudaSuccess ||
        (e = cudaMalloc((void**)&p.snap_id, (size_t)p.cap_pad * 4)) != cudaSuccess ||
        (e = cudaMalloc((void**)&p.snap_off, (size_t)(kSnapBins + 1) * 4)) != cudaSuccess ||
        (e = cudaMalloc((void**)&p.snap_aux, (size_t)(kSnapBins + 4) * 4)) != cudaSuccess)
      return e;
  }
  uint32_t* aux = p.snap_aux;
  if ((e = cudaMemsetAsync(aux, 0, (size_t)(kSnapBins + 2) * 4, s)) != cudaSuccess ||
      (e = cudaMemsetAsync(aux + kSnapBins, 0xFF, 4, s)) != cudaSuccess)
    return e;
  const int grid = 4 * p.num_sms;
  snap_minmax_kernel<<<grid, 256, 0, s>>>(p.joints, L, p.JP, aux + kSnapBins);
  snap_hist_kernel<<<grid, 256, 0, s>>>(p.joints, L, p.JP, aux);
  snap_scan_kernel<<<1, 1024, 0, s>>>(aux, p.snap_off);
  snap_scatter_kernel<<<grid, 256, 0, s>>>(p.joints, L, p.JP, aux, p.snap_j, p.snap_id);
  p.launches += 4;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  p.snap_L = L;
  return cudaSuccess;
}

// gate-first kernels are programmatic dependents of the kernel before them (query prep,
// then the gate scan): each starts with griddep_wait()
inline cudaLaunchConfig_t gf_config(dim3 grid, int threads, cudaStream_t s, cudaLaunchAttribute* attr) {
  return pdl_config(grid, dim3(threads), 0, s, attr);
}

// One gate-scan launch over `tiles` joint tiles with QT queries per block: ~2 full waves
// of resident blocks, but >= 8 tiles per block so per-block setup stays amortised.
// (Resident blocks per SM depend only on the kernel and the device: cached on the pool.)
template <int JP, int QT>
cudaError_t launch_gate_scan(Pool& p, const MatchArgs& a, int32_t cap, const GfRows& rows, int64_t tiles,
                             int32_t sorted, cudaStream_t s) {
  int& occ = p.gf_occ[JP == 4 ? 0 : JP == 8 ? 1 : 2][QT == 32 ? 0 : QT == 64 ? 1 : QT == 128 ? 2 : 3];
  if (occ == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gate_scan_kernel<JP, QT>, kGfThreads, 0);
    if (e != cudaSuccess) return e;
    occ = std::max(occ, 1);
  }
  const int n_qg = (a.nq + QT - 1) / QT;
  const int S = (int)std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(1, tiles / 8),
                                                            (2 * (int64_t)occ * p.num_sms + n_qg - 1) / n_qg));
  cudaLaunchAttribute attr[1];
  const cudaLaunchConfig_t cfg = gf_config(dim3(n_qg, S), kGfThreads, s, attr);
  ++p.launches;
  return cudaLaunchKernelEx(&cfg, gate_scan_kernel<JP, QT>, rows, static_cast<const float*>(p.q_joints), a.nq, S,
                            a.g2, cap, p.gf_cnt, p.gf_cand, sorted);
}

template <int JP>
cudaError_t launch_gate_scan_q(Pool& p, const MatchArgs& a, int32_t cap, const GfRows& rows, int64_t tiles,
                               int32_t sorted, cudaStream_t s) {
  // queries per block: the batch rounded up to a power-of-two warp multiple; the other
  // warps split the rows (C5 pool, 64 queries: 340 us with 256 queries per block)
  if (a.nq <= 32) return launch_gate_scan<JP, 32>(p, a, cap, rows, tiles, sorted, s);
  if (a.nq <= 64) return launch_gate_scan<JP, 64>(p, a, cap, rows, tiles, sorted, s);
  if (a.nq <= 128) return launch_gate_scan<JP, 128>(p, a, cap, rows, tiles, sorted, s);
  return launch_gate_scan<JP, kGfThreads>(p, a, cap, rows, tiles, sorted, s);
}

template <int JP>
cudaError_t launch_gf_jp(Pool& p, const MatchArgs& a, int32_t cap, float* out_s, int64_t* out_i, uint8_t* out_hit,
                         bool sorted, cudaStream_t s) {
  const int64_t n_pt = (p.local + kGfTile - 1) / kGfTile;
  cudaError_t e = cudaSuccess;
  if (!a.zeroed && (e = cudaMemsetAsync(p.gf_cnt, 0, (size_t)a.nq * sizeof(uint32_t), s)) != cudaSuccess) return e;
  // Sorted batches on large pools scan the joint-0 index: each block of queries visits
  // only the rows within gamma of its joint-0 interval (plus the unsorted tail).
  const bool snap = sorted && !a.qbins && p.local >= kSnapMinRows;
  if (snap && (e = snap_refresh(p, s)) != cudaSuccess) return e;
  const int64_t plain_begin = snap ? p.snap_L : 0;
  if (snap) {
    const GfRows rows{p.snap_j, p.snap_id, 0, p.snap_L, p.snap_off,
                      reinterpret_cast<const float*>(p.snap_aux + kSnapBins + 2)};
    if ((e = launch_gate_scan_q<JP>(p, a, cap, rows, n_pt, 1, s)) != cudaSuccess) return e;
  }
  if (a.qbins && p.local > 0) {
    // 17..1024 gated queries in joint-0 bins: pools of >= 64 K rows scan their joint-0
    // snapshot with warp-uniform windows, the rows appended since (or a small pool) with
    // the pair-dealing kernel
    const bool use_snap = p.local >= kSnapMinRows;
    if (use_snap && (e = snap_refresh(p, s)) != cudaSuccess) return e;
    const int64_t tail = use_snap ? p.snap_L : 0;
    const size_t smem = (size_t)a.nq * (JP + 1) * 4 + (size_t)(kQBins + 1) * 4;
    size_t& opted = p.gf_rows_smem_opt;   // dynamic shared memory above 48 KB needs the opt-in (once per pool)
    if (smem > opted) {
      if ((e = cudaFuncSetAttribute(gate_rows_binned_kernel<JP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem)) != cudaSuccess ||
          (e = cudaFuncSetAttribute(gate_rows_snap_kernel<JP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem)) != cudaSuccess)
        return e;
      opted = smem;
    }
    cudaLaunchAttribute attr[1];
    if (use_snap) {
      const unsigned grid = (unsigned)std::max<int64_t>(
          1, std::min<int64_t>((tail + kGfRowsThreads - 1) / kGfRowsThreads, 8 * (int64_t)p.num_sms));
      cudaLaunchConfig_t cfg = gf_config(dim3(grid), kGfRowsThreads, s, attr);
      cfg.dynamicSmemBytes = smem;
      ++p.launches;
      if ((e = cudaLaunchKernelEx(&cfg, gate_rows_snap_kernel<JP>, static_cast<const float*>(p.snap_j),
                                  static_cast<const int32_t*>(p.snap_id), tail, static_cast<const float*>(p.q_joints),
                                  a.nq, a.g2, cap, p.gf_cnt, p.gf_cand, static_cast<const int32_t*>(p.gf_qbins))) !=
          cudaSuccess)
        return e;
    }
    if (p.local > tail) {
      const unsigned grid = (unsigned)std::max<int64_t>(
          1, std::min<int64_t>((p.local - tail + kGfRowsThreads - 1) / kGfRowsThreads, 8 * (int64_t)p.num_sms));
      cudaLaunchConfig_t cfg = gf_config(dim3(grid), kGfRowsThreads, s, attr);
      cfg.dynamicSmemBytes = smem;
      ++p.launches;
      if ((e = cudaLaunchKernelEx(&cfg, gate_rows_binned_kernel<JP>, static_cast<const float*>(p.joints), tail,
                                  p.local, static_cast<const float*>(p.q_joints), a.nq, a.g2, cap, p.gf_cnt,
                                  p.gf_cand, static_cast<const int32_t*>(p.gf_qbins))) != cudaSuccess)
        return e;
    }
  } else if (p.local > plain_begin && plain_begin == 0 && a.nq <= kGfRowsMaxQ) {
    // tiny batch over the whole pool: the row-parallel kernel (~2 waves of 8 blocks per SM)
    const unsigned grid = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((p.local + kGfRowsThreads - 1) / kGfRowsThreads, 16 * (int64_t)p.num_sms));
    cudaLaunchAttribute attr[1];
    const cudaLaunchConfig_t cfg = gf_config(dim3(grid), kGfRowsThreads, s, attr);
    ++p.launches;
    if ((e = cudaLaunchKernelEx(&cfg, gate_rows_kernel<JP>, static_cast<const float*>(p.joints), p.local,
                                static_cast<const float*>(p.q_joints), a.nq, a.g2, cap, p.gf_cnt, p.gf_cand)) !=
        cudaSuccess)
      return e;
  } else if (p.local > plain_begin) {
    const int64_t tail_tiles = (p.local + kGfTile - 1) / kGfTile - plain_begin / kGfTile;
    const GfRows rows{p.joints, nullptr, plain_begin, p.local, nullptr, nullptr};
    if ((e = launch_gate_scan_q<JP>(p, a, cap, rows, tail_tiles, sorted ? 1 : 0, s)) != cudaSuccess) return e;
  }
  const int wpb = 4;
  const unsigned g = (unsigned)((a.nq + wpb - 1) / wpb);
  const auto& c = p.cfg;
  cudaLaunchAttribute attr[1];
  const cudaLaunchConfig_t cfg = gf_config(dim3(g), wpb * 32, s, attr);
#define AMS_GF(KT_)                                                                                           \
  e = cudaLaunchKernelEx(&cfg, score_kernel<KT_, JP>, static_cast<const uint16_t*>(p.emb),                    \
                         static_cast<const float*>(p.inv_norm), static_cast<const float*>(p.joints), p.local,   \
                         static_cast<const uint16_t*>(p.q_stage), static_cast<const float*>(p.q_inv),           \
                         static_cast<const float*>(p.q_joints), c.dim, a.nq, a.k, a.g2, cap,                   \
                         static_cast<const uint32_t*>(p.gf_cnt), static_cast<const int32_t*>(p.gf_cand), out_s, \
                         out_i, out_hit, a.threshold, c.rank, c.world, p.B,                                    \
                         static_cast<const int32_t*>(sorted ? p.q_perm : nullptr))
  switch (a.KT) {
    case 8: AMS_GF(8); break;
    case 16: AMS_GF(16); break;
    case 32: AMS_GF(32); break;
    default: AMS_GF(64); break;
  }
#undef AMS_GF
  ++p.launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Pass-rate estimate for ams_match_auto: exact canonical gate over a strided sample of
// up to kEstQueries queries (raw [nq][J] joints) x up to kEstRows local rows; out[0] +=
// eligible sampled pairs.  Thread per sampled row, loop over the sampled queries.
__global__ void gate_estimate_kernel(const float* __restrict__ pool_joints, int32_t JP, int64_t L, int64_t row_step,
                                     int32_t n_rows, const float* __restrict__ qj, int32_t J, int32_t q_step,
                                     int32_t n_q, float g2, unsigned long long* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned int c = 0;
  if (r < n_rows) {
    const int64_t l = (int64_t)r * row_step;
    float pj[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) pj[t] = t < J ? pool_joints[joint_offset(l, t, JP)] : 0.0f;
    for (int i = 0; i < n_q; ++i) {
      const float* q = qj + (int64_t)i * q_step * J;
      float ds = 0.0f;
#pragma unroll
      for (int t = 0; t < 16; ++t)
        if (t < J) {
          const float diff = q[t] - pj[t];
          ds = fmaf(diff, diff, ds);
        }
      c += ds <= g2 ? 1u : 0u;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

}  // namespace

cudaError_t launch_gate_estimate(Pool& p, const float* qj_raw, int32_t nq, float g2, unsigned long long* out,
                                 int32_t* rows_sampled, int32_t* queries_sampled, cudaStream_t s) {
  const int64_t L = p.local;
  const int64_t row_step = std::max<int64_t>(1, (L + kEstRows - 1) / kEstRows);
  const int32_t n_rows = (int32_t)((L + row_step - 1) / row_step);
  const int32_t q_step = std::max<int32_t>(1, (nq + kEstQueries - 1) / kEstQueries);
  const int32_t n_q = (nq + q_step - 1) / q_step;
  *rows_sampled = n_rows;
  *queries_sampled = n_q;
  cudaError_t e = cudaMemsetAsync(out, 0, 8, s);
  if (e != cudaSuccess || n_rows == 0) return e;
  gate_estimate_kernel<<<(n_rows + 255) / 256, 256, 0, s>>>(p.joints, p.JP, L, row_step, n_rows, qj_raw,
                                                            p.cfg.joint_dim, q_step, n_q, g2, out);
  ++p.launches;
  return cudaGetLastError();
}

cudaError_t launch_query_order_j0(Pool& p, const float* qj_src, int32_t nq, cudaStream_t s) {
  query_order_j0_kernel<<<1, kQOrderThreads, 0, s>>>(qj_src, p.cfg.joint_dim, nq, p.q_perm, p.gf_qbins);
  ++p.launches;
  return cudaGetLastError();
}

cudaError_t launch_gate_first(Pool& p, const MatchArgs& a, float* out_s, int64_t* out_i, uint8_t* out_hit,
                              bool sorted, cudaStream_t s) {
  const int32_t cap = p.gf_cap;
  switch (p.JP) {
    case 4: return launch_gf_jp<4>(p, a, cap, out_s, out_i, out_hit, sorted, s);
    case 8: return launch_gf_jp<8>(p, a, cap, out_s, out_i, out_hit, sorted, s);
    default: return launch_gf_jp<16>(p, a, cap, out_s, out_i, out_hit, sorted, s);
  }
}

}  // namespace ams
