// ams_match_tc.cu -- tcgen05/TMEM/TMA similarity GEMM with the fused gate + top-k
// epilogue (bf16 pools).  The score matrix never reaches HBM.
//
// Method (3.2.1 "comparing the similarity"; north_star metric):
//   acc(i,j)  = sum_t q_it * e_jt          bf16 x bf16 -> fp32 on the tensor cores
//   s(i,j)    = (acc * inv_q_i) * inv_e_j  fp32
//   gate(i,j) = canonical fp32 sum_t (r_it - p_jt)^2 <= g2
//   top-k by (s desc, j asc) per query, kept in registers of the epilogue threads.
//
// Tiling: a tile is 128 queries (TMEM lanes, MMA M) x 256 pool rows (TMEM columns,
// MMA N); K advances 64 bf16 (one 128-B swizzle atom) per pipeline stage, 4 UMMAs of
// K=16 per stage.  A work unit is (query tile, contiguous split of the pool rows); a
// persistent CTA walks its units in split-major order so concurrent CTAs share the
// same pool rows through L2.
//
// Warp roles (320 threads, 1 CTA / SM):
//   warp 0      TMA producer: query + pool tiles into a STAGES-deep smem ring; pool
//               joints / inv_norm of each tile into a 2-deep aux ring (bulk copies)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer; accumulators
//               double-buffered in TMEM (2 x 256 columns)
//   warps 2..9  epilogue: warp w reads TMEM lanes 32*(w%4).. (its 32 queries), column
//               half (w-2)/4 of the tile, with tcgen05.ld; scales, gates, keeps a
//               per-thread running top-k; one partial list per (query, split, half).
#include <cuda_bf16.h>
#include <math_constants.h>

#include "ams_internal.cuh"
#include "ams_ptx.cuh"
#include "ams_topk.cuh"

namespace ams {

namespace {

constexpr int kThreadsTc = 64 + 128 * kEpiHalves;   // 320
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kABytes = kBlockM * kBlockK * 2;   // 16 KB
constexpr uint32_t kBBytes = kBlockN * kBlockK * 2;   // 32 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(kBlockM, kBlockN);
constexpr int kColsPerHalf = kBlockN / kEpiHalves;    // 128
constexpr int kChunk = 32;

struct TcParams {
  const float* inv_q;
  const float* q_joints;     // [q_pad, JP]
  const float* pool_inv;     // [cap_pad]
  const float* pool_joints;  // [cap_pad, JP]
  float* part_s;
  int32_t* part_i;
  int64_t L;                 // local rows
  int32_t nq, d, n_qt, n_pt, S, n_units, k, gated, P;
  float g2;
};

template <int JP>
struct SmemLayout {
  static constexpr uint32_t aux_j_bytes = kBlockN * JP * 4;
  static constexpr uint32_t aux_bytes = aux_j_bytes + kBlockN * 4;
};

__host__ __device__ constexpr int stages_for(int JP) { return JP >= 16 ? 3 : 4; }

template <int JP>
__host__ __device__ constexpr size_t smem_for() {
  return 1024 /*align slack*/ + (size_t)stages_for(JP) * kStageBytes + 2 * SmemLayout<JP>::aux_bytes + 256;
}

__device__ __forceinline__ void split_tiles(int sp, int S, int n_pt, int& t_lo, int& t_hi) {
  t_lo = (int)((int64_t)sp * n_pt / S);
  t_hi = (int)((int64_t)(sp + 1) * n_pt / S);
}

template <int KT, int JP, bool GATED>
__device__ __forceinline__ void epi_chunk(const uint32_t (&v)[32], uint32_t taddr, int64_t jbase,
                                          int64_t row_end, const float* __restrict__ inv_e_sm,
                                          const float* __restrict__ joints_sm, const float (&qj)[JP], float iq,
                                          float g2, int k, TopK<KT, int32_t>& top) {
  uint32_t m = 0;
#pragma unroll
  for (int c = 0; c < kChunk; c += 4) {
    const float4 ie = *reinterpret_cast<const float4*>(inv_e_sm + c);
    const float iev[4] = {ie.x, ie.y, ie.z, ie.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int cc = c + u;
      const float s = __fmul_rn(__fmul_rn(__uint_as_float(v[cc]), iq), iev[u]);
      bool cand = (s > top.kth_s) && (jbase + cc < row_end);
      if (GATED) {
        const float4* pj = reinterpret_cast<const float4*>(joints_sm + cc * JP);
        float4 p = pj[0];
        float df = __fsub_rn(qj[0], p.x);
        float ds = __fmaf_rn(df, df, 0.0f);
        df = __fsub_rn(qj[1], p.y);
        ds = __fmaf_rn(df, df, ds);
        df = __fsub_rn(qj[2], p.z);
        ds = __fmaf_rn(df, df, ds);
        df = __fsub_rn(qj[3], p.w);
        ds = __fmaf_rn(df, df, ds);
        cand = cand && (ds <= g2);
        if (JP > 4) {
          if (__any_sync(0xffffffffu, cand)) {
#pragma unroll
            for (int g = 1; g < JP / 4; ++g) {
              p = pj[g];
              df = __fsub_rn(qj[4 * g + 0], p.x);
              ds = __fmaf_rn(df, df, ds);
              df = __fsub_rn(qj[4 * g + 1], p.y);
              ds = __fmaf_rn(df, df, ds);
              df = __fsub_rn(qj[4 * g + 2], p.z);
              ds = __fmaf_rn(df, df, ds);
              df = __fsub_rn(qj[4 * g + 3], p.w);
              ds = __fmaf_rn(df, df, ds);
              cand = cand && (ds <= g2);
              if (!__any_sync(0xffffffffu, cand)) break;
            }
          }
        }
      }
      m |= (cand ? 1u : 0u) << cc;
    }
  }
  // rare path: insert candidates; re-read the accumulator column (warp-uniform loop,
  // tcgen05.ld is warp-collective) and recompute the identical score.
  uint32_t wm = __reduce_or_sync(0xffffffffu, m);
  while (wm != 0u) {
    const int c = __ffs(wm) - 1;
    wm &= wm - 1u;
    const uint32_t raw = ptx::tmem_ld1(taddr + (uint32_t)c);
    ptx::tmem_wait_ld();
    if ((m >> c) & 1u) {
      const float s = __fmul_rn(__fmul_rn(__uint_as_float(raw), iq), inv_e_sm[c]);
      if (s > top.kth_s) top.insert_monotone(s, (int32_t)(jbase + c), k);
    }
  }
}

template <int KT, int JP>
__global__ void __launch_bounds__(kThreadsTc, 1)
    match_tc_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_pool,
                    const TcParams prm) {
  constexpr int STAGES = stages_for(JP);
  constexpr uint32_t AUXJ = SmemLayout<JP>::aux_j_bytes;
  constexpr uint32_t AUX = SmemLayout<JP>::aux_bytes;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                   // STAGES x 16 KB
  uint8_t* sB = smem + STAGES * kABytes;                // STAGES x 32 KB
  uint8_t* sAux = smem + STAGES * kStageBytes;          // 2 x AUX
  uint64_t* bars = reinterpret_cast<uint64_t*>(sAux + 2 * AUX);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* afull = tfull + 4;
  uint64_t* aempty = tfull + 6;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tfull + 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_q);
    ptx::prefetch_tmap(&tmap_pool);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 4 * kEpiHalves);
      ptx::mbar_init(&afull[i], 1);
      ptx::mbar_init(&aempty[i], 4 * kEpiHalves);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(tmem_holder, kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int n_kb = prm.d / kBlockK;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol_q = ptx::policy_evict_last();
      const uint64_t pol_pool = prm.n_qt > 1 ? ptx::policy_evict_normal() : ptx::policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      uint32_t tile_count = 0;
      for (int u = blockIdx.x; u < prm.n_units; u += gridDim.x) {
        const int sp = u / prm.n_qt, qt = u % prm.n_qt;
        int t_lo, t_hi;
        split_tiles(sp, prm.S, prm.n_pt, t_lo, t_hi);
        for (int t = t_lo; t < t_hi; ++t, ++tile_count) {
          const int buf = tile_count & 1;
          const uint32_t use = tile_count >> 1;
          ptx::mbar_wait(&aempty[buf], (use & 1u) ^ 1u);
          uint8_t* aux = sAux + buf * AUX;
          ptx::mbar_arrive_expect_tx(&afull[buf], AUX);
          ptx::bulk_load(aux, prm.pool_joints + (int64_t)t * kBlockN * JP, AUXJ, &afull[buf]);
          ptx::bulk_load(aux + AUXJ, prm.pool_inv + (int64_t)t * kBlockN, kBlockN * 4, &afull[buf]);
          for (int kb = 0; kb < n_kb; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1u);
            ptx::mbar_arrive_expect_tx(&full[stage], kStageBytes);
            ptx::tma_load_2d(sA + stage * kABytes, &tmap_q, &full[stage], kb * kBlockK, qt * kBlockM, pol_q);
            ptx::tma_load_2d(sB + stage * kBBytes, &tmap_pool, &full[stage], kb * kBlockK, t * kBlockN,
                             pol_pool);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t tile_count = 0;
      for (int u = blockIdx.x; u < prm.n_units; u += gridDim.x) {
        const int sp = u / prm.n_qt;
        int t_lo, t_hi;
        split_tiles(sp, prm.S, prm.n_pt, t_lo, t_hi);
        for (int t = t_lo; t < t_hi; ++t, ++tile_count) {
          const int buf = tile_count & 1;
          const uint32_t use = tile_count >> 1;
          ptx::mbar_wait(&tempty[buf], (use & 1u) ^ 1u);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(buf * kBlockN);
          for (int kb = 0; kb < n_kb; ++kb) {
            ptx::mbar_wait(&full[stage], phase);
            ptx::tc_fence_after();
            const uint32_t a0 = ptx::smem_u32(sA + stage * kABytes);
            const uint32_t b0 = ptx::smem_u32(sB + stage * kBBytes);
#pragma unroll
            for (int kk = 0; kk < kBlockK / 16; ++kk) {
              ptx::umma_f16(d_tmem, ptx::sdesc_k_sw128(a0 + kk * 32), ptx::sdesc_k_sw128(b0 + kk * 32), kIdesc,
                            (kb | kk) != 0 ? 1u : 0u);
            }
            ptx::umma_commit(&empty[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
          ptx::umma_commit(&tfull[buf]);
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int e = warp - 2;
    const int lg = warp & 3;           // TMEM lane group accessible to this warp
    const int h = e >> 2;              // column half
    uint32_t tile_count = 0;
    const bool gated = prm.gated != 0;
    for (int u = blockIdx.x; u < prm.n_units; u += gridDim.x) {
      const int sp = u / prm.n_qt, qt = u % prm.n_qt;
      int t_lo, t_hi;
      split_tiles(sp, prm.S, prm.n_pt, t_lo, t_hi);
      const int64_t row_end = min((int64_t)t_hi * kBlockN, prm.L);
      const int qrow = qt * kBlockM + lg * 32 + lane;
      const bool active = qrow < prm.nq;
      float qj[JP];
      float iq = 0.0f;
#pragma unroll
      for (int t = 0; t < JP; ++t) qj[t] = active ? prm.q_joints[(int64_t)qrow * JP + t] : 0.0f;
      if (active) iq = prm.inv_q[qrow];
      TopK<KT, int32_t> top;
      top.init(active);
      for (int t = t_lo; t < t_hi; ++t, ++tile_count) {
        const int buf = tile_count & 1;
        const uint32_t use = tile_count >> 1;
        ptx::mbar_wait(&afull[buf], use & 1u);
        ptx::mbar_wait(&tfull[buf], use & 1u);
        ptx::tc_fence_after();
        const uint8_t* aux = sAux + buf * AUX;
        const float* joints_sm = reinterpret_cast<const float*>(aux);
        const float* inv_sm = reinterpret_cast<const float*>(aux + AUXJ);
#pragma unroll 1
        for (int ch = 0; ch < kColsPerHalf / kChunk; ++ch) {
          const int col0 = h * kColsPerHalf + ch * kChunk;
          const uint32_t taddr = tmem_base + ((uint32_t)(lg * 32) << 16) + (uint32_t)(buf * kBlockN + col0);
          uint32_t v[32];
          ptx::tmem_ld32(taddr, v);
          ptx::tmem_wait_ld();
          const int64_t jbase = (int64_t)t * kBlockN + col0;
          if (gated)
            epi_chunk<KT, JP, true>(v, taddr, jbase, row_end, inv_sm + col0, joints_sm + col0 * JP, qj, iq,
                                    prm.g2, prm.k, top);
          else
            epi_chunk<KT, JP, false>(v, taddr, jbase, row_end, inv_sm + col0, joints_sm + col0 * JP, qj, iq,
                                     prm.g2, prm.k, top);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&tempty[buf]);
          ptx::mbar_arrive(&aempty[buf]);
        }
      }
      if (active) {
        const int64_t base = ((int64_t)qrow * prm.P + (int64_t)sp * kEpiHalves + h) * KT;
#pragma unroll
        for (int r = 0; r < KT; r += 4) {
          *reinterpret_cast<float4*>(prm.part_s + base + r) = make_float4(top.s[r], top.s[r + 1], top.s[r + 2], top.s[r + 3]);
          *reinterpret_cast<int4*>(prm.part_i + base + r) = make_int4(top.i[r], top.i[r + 1], top.i[r + 2], top.i[r + 3]);
        }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, kTmemCols);
  }
}

template <int KT, int JP>
cudaError_t launch_tc_t(Pool& p, const TcParams& prm, int grid, cudaStream_t s) {
  auto kern = match_tc_kernel<KT, JP>;
  const size_t smem = smem_for<JP>();
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  kern<<<grid, kThreadsTc, smem, s>>>(p.tmap_q, p.tmap_pool, prm);
  return cudaGetLastError();
}

template <int KT>
cudaError_t launch_tc_kt(Pool& p, const TcParams& prm, int grid, cudaStream_t s) {
  switch (p.JP) {
    case 4: return launch_tc_t<KT, 4>(p, prm, grid, s);
    case 8: return launch_tc_t<KT, 8>(p, prm, grid, s);
    default: return launch_tc_t<KT, 16>(p, prm, grid, s);
  }
}

}  // namespace

int tc_stages(int JP) { return stages_for(JP); }
size_t tc_smem_bytes(int JP) {
  return JP <= 4 ? smem_for<4>() : JP <= 8 ? smem_for<8>() : smem_for<16>();
}

cudaError_t launch_match_tc(Pool& p, const MatchArgs& a, int32_t S, int32_t grid, cudaStream_t s) {
  TcParams prm{};
  prm.inv_q = p.q_inv;
  prm.q_joints = p.q_joints;
  prm.pool_inv = p.inv_norm;
  prm.pool_joints = p.joints;
  prm.part_s = p.part_s;
  prm.part_i = p.part_i;
  prm.L = p.local;
  prm.nq = a.nq;
  prm.d = p.cfg.dim;
  prm.n_qt = (a.nq + kBlockM - 1) / kBlockM;
  prm.n_pt = (int32_t)((p.local + kBlockN - 1) / kBlockN);
  prm.S = S;
  prm.n_units = prm.n_qt * S;
  prm.k = a.k;
  prm.gated = a.gated;
  prm.P = S * kEpiHalves;
  prm.g2 = a.g2;
  cudaError_t e;
  switch (a.KT) {
    case 8: e = launch_tc_kt<8>(p, prm, grid, s); break;
    case 16: e = launch_tc_kt<16>(p, prm, grid, s); break;
    case 32: e = launch_tc_kt<32>(p, prm, grid, s); break;
    default: e = launch_tc_kt<64>(p, prm, grid, s); break;
  }
  ++p.launches;
  return e;
}

}  // namespace ams
