// ams_match_tc.cu -- tcgen05/TMEM/TMA similarity GEMM with the fused gate + top-k
// epilogue (bf16 pools).  The score matrix never reaches HBM.
//
// Method (3.2.1 "comparing the similarity"; north_star metric):
//   acc(i,j)  = sum_t q_it * e_jt          bf16 x bf16 -> fp32 on the tensor cores
//   s(i,j)    = (acc * inv_q_i) * inv_e_j  fp32
//   gate(i,j) = canonical fp32 sum_t (r_it - p_jt)^2 <= g2
//   top-k by (s desc, j asc) per query, kept in registers of the epilogue threads.
//
// Tiling: a tile is 128*CG queries (MMA M; TMEM lanes of each CTA) x 256 pool rows
// (MMA N; TMEM columns); K advances 64 bf16 (one 128-B swizzle atom) per pipeline
// stage, 4 UMMAs of K=16 per stage.  CG = 2 runs the tile on a CTA pair
// (tcgen05.mma.cta_group::2, M = 256): each CTA stages its own 128 query rows and half
// of the 256 pool rows, so a pair tile moves 1 MB of operands per 134 MFLOP (128 flop/B
// from L2, vs 85 for the single-CTA 128x256 tile).  A work unit is (query tile,
// contiguous split of the pool rows); persistent clusters walk units in split-major
// order so concurrent CTAs stream the same pool rows through L2.
//
// Warp roles (320 threads per CTA, 1 CTA per SM).  The warp scheduler issues the
// highest warp id first, so the two latency-critical single-thread roles take the top
// ids and are never queued behind epilogue math on their sub-partition:
//   warps 0..7  epilogue: warp w reads TMEM lanes 32*(w%4).. (its 32 queries) of column
//               half w/4 with tcgen05.ld; one partial list per (query, split, half).
//   warp 8      TMA producer: query + pool tiles into a STAGES-deep smem ring; pool
//               joints / inv_norm of each tile into a 2-deep aux ring (bulk copies)
//   warp 9      TMEM allocator + (leader CTA) single-thread tcgen05.mma issuer;
//               accumulators double-buffered in TMEM (2 x 256 columns)
//
// Epilogue per 32-column chunk: a branch-free filter computes, with packed f32x2
// math, either the chunk's best score (ungated) or the smallest partial joint distance
// over the first 4 joints (gated; partial sums of squares are a lower bound of the
// canonical sum since RN is monotone), then ONE warp vote decides whether the exact
// per-column path runs.  Admission uses the local KT-th best AND a per-query lower bound
// shared through global memory by every split of the same query (the KT-th best of any
// split is <= the global k-th best, so rows below it can never enter; equal scores are
// admitted so the index tie rule is preserved).
#include <cuda_bf16.h>
#include <math_constants.h>

#include "ams_internal.cuh"
#include "ams_ptx.cuh"
#include "ams_topk.cuh"

namespace ams {

namespace {

constexpr int kThreadsTc = 64 + 128 * kEpiHalves;   // 320
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kABytes = kBlockM * kBlockK * 2;   // 16 KB: 128 query rows x 128 B
constexpr int kColsPerHalf = kBlockN / kEpiHalves;    // 128
constexpr int kChunk = 32;

template <int CG>
struct Geo {
  static constexpr uint32_t b_rows = kBlockN / CG;               // pool rows staged per CTA
  static constexpr uint32_t b_bytes = b_rows * kBlockK * 2;      // 32 KB (CG 1) / 16 KB (CG 2)
  static constexpr uint32_t stage_bytes = kABytes + b_bytes;
  static constexpr uint32_t idesc = ptx::idesc_bf16_f32(kBlockM * CG, kBlockN);
};

struct TcParams {
  const float* inv_q;
  const float* q_joints;     // [q_pad, JP]
  const float* pool_inv;     // [cap_pad]
  const float* pool_joints;  // [cap_pad/256][JP][256]
  float* part_s;
  int32_t* part_i;
  uint32_t* bound;           // [nq] per-query admission lower bound (ordered-u32; 0 = none)
  uint32_t* wave_ctr;        // producers' unit-completion counter (zeroed per launch; bound[nq])
  const int32_t* perm;       // staged query position -> caller's query (nullptr: identity)
  uint32_t* slots;           // [q_pad][KT] union-bound slots (ordered-u32; ungated only, else null)
  int64_t L;                 // local rows
  int32_t nq, d, n_qt, n_pt, S, n_units, k, gated, P;
  int32_t sorted;            // queries staged in (joint 0, joint 1) order: the warp-level column test pays
  float g2;
};

template <int JP>
struct Aux {
  static constexpr uint32_t j_bytes = kBlockN * JP * 4;
  static constexpr uint32_t bytes = j_bytes + kBlockN * 4;
};

// Per-tile joints / inverse norms ring.  Three deep: the producer loads tile t+1's aux
// before its k-blocks, and with two buffers it waited for the epilogue of tile t-1,
// which only starts when the MMA of t-1 ends -- a slow epilogue then starved the MMA.
constexpr int kAuxDepth = 3;

template <int JP, int CG>
__host__ __device__ constexpr int stages_for() {
  return CG == 1 ? (JP >= 16 ? 3 : 4) : (JP >= 16 ? 5 : 6);
}

template <int JP, int CG>
__host__ __device__ constexpr size_t smem_for() {
  return 1024 /*align slack*/ + (size_t)stages_for<JP, CG>() * Geo<CG>::stage_bytes + kAuxDepth * Aux<JP>::bytes + 256;
}

__device__ __forceinline__ void split_tiles(int sp, int S, int n_pt, int& t_lo, int& t_hi) {
  t_lo = (int)((int64_t)sp * n_pt / S);
  t_hi = (int)((int64_t)(sp + 1) * n_pt / S);
}

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// One 32-column chunk of the epilogue for one thread (= one query).
//   inv_sm: inverse norms of the chunk's 32 pool rows (smem)
//   jsm:    joint t of chunk column c at jsm[t * 256 + c] (smem, tile-transposed)
// Fast filter: one value per 8-column sub-chunk (best score, or smallest partial joint
// distance); the exact path reloads only sub-chunks that some lane may admit.
template <int KT, int JP, bool GATED>
__device__ __forceinline__ void epi_chunk(uint32_t taddr, int64_t jbase, int nvalid,
                                          const float* __restrict__ inv_sm, const float* __restrict__ jsm,
                                          const uint64_t (&QQ)[4], const float (&qj)[JP], float iq, float ie_min,
                                          float ie_max, float g2, float bound, int k, TopK<KT, int32_t>& top) {
  constexpr int JF = JP < 4 ? JP : 4;   // joints in the filter
  uint32_t fire = 0;                    // bit sub: some column of sub-chunk sub may be admitted
  if (GATED) {
#pragma unroll
    for (int sub = 0; sub < 4; ++sub) {
      float mn = CUDART_INF_F;
#pragma unroll
      for (int c4 = 2 * sub; c4 < 2 * sub + 2; ++c4) {
        uint64_t da = 0ull, db = 0ull;   // +0.0f pairs
#pragma unroll
        for (int t = 0; t < JF; ++t) {
          const float4 p = lds4(jsm + t * kBlockN + 4 * c4);
          const uint64_t a = ptx::sub2(QQ[t], ptx::pack2(p.x, p.y));
          da = ptx::fma2(a, a, da);
          const uint64_t b = ptx::sub2(QQ[t], ptx::pack2(p.z, p.w));
          db = ptx::fma2(b, b, db);
        }
        mn = fminf(mn, fminf(fminf(ptx::lo2(da), ptx::hi2(da)), fminf(ptx::lo2(db), ptx::hi2(db))));
      }
      fire |= (mn <= g2 ? 1u : 0u) << sub;
    }
  } else {
    // Upper bound of the 8 scores of a sub-chunk from the raw maximum: with
    // m = RN(max_c acc_c * iq), every s_c = RN(RN(acc_c * iq) * ie_c) is <= RN(m * ie_max)
    // when m >= 0 and <= RN(m * ie_min) when m < 0 (iq, ie >= 0; RN is monotone), where
    // ie_min/ie_max bound the tile's inverse norms.  0.5 FMNMX3 per column instead of
    // scaling every score.
    uint32_t v[32];
    __syncwarp();
    ptx::tmem_ld32(taddr, v);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int sub = 0; sub < 4; ++sub) {
#define AMS_V(c) __uint_as_float(v[8 * sub + (c)])
      const float mv = fmaxf(ptx::fmax3(ptx::fmax3(AMS_V(0), AMS_V(1), AMS_V(2)), ptx::fmax3(AMS_V(3), AMS_V(4), AMS_V(5)),
                                        AMS_V(6)),
                             AMS_V(7));
#undef AMS_V
      const float m = __fmul_rn(mv, iq);
      const float ub = __fmul_rn(m, m >= 0.0f ? ie_max : ie_min);
      fire |= (ub > top.kth_s && ub >= bound ? 1u : 0u) << sub;
    }
  }
  uint32_t wfire = __reduce_or_sync(0xffffffffu, fire);
  // exact path (rare), sub-chunk by sub-chunk; tcgen05.ld is warp-collective and the
  // loop is warp-uniform
  while (wfire != 0u) {
    const int sub = __ffs(wfire) - 1;
    wfire &= wfire - 1u;
    __syncwarp();   // tcgen05.ld is .sync.aligned: reconverge after the previous inserts
    uint32_t v8[8];
    ptx::tmem_ld8(taddr + (uint32_t)(sub * 8), v8);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int cc = sub * 8 + c;
      const float s = __fmul_rn(__fmul_rn(__uint_as_float(v8[c]), iq), inv_sm[cc]);
      bool ok = (s > top.kth_s) && (s >= bound) && (cc < nvalid);
      if (GATED) {
        float ds = 0.0f;
#pragma unroll
        for (int g = 0; g < JP / 4; ++g) {
          if (!__any_sync(0xffffffffu, ok)) break;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float df = __fsub_rn(qj[4 * g + u], jsm[(4 * g + u) * kBlockN + cc]);
            ds = __fmaf_rn(df, df, ds);
          }
          ok = ok && (ds <= g2);
        }
      }
      if (ok) top.insert_monotone(s, (int32_t)(jbase + cc), k);
    }
  }
}

// Gated chunk for a warp whose 32 queries are ordered by (joint 0, joint 1) (their r_0
// lie in [wlo, whi], r_1 in [wlo1, whi1]).  Lane c first tests column c against the
// whole warp at once: the canonical distance after two joints is
// fmaf(d1, d1, RN(d0^2)) and later terms only add (RN is monotone); |RN(r_t - p_t)| is
// smallest at the interval end nearer to p_t, so with D_t = RN(w_t - p_t) for that end
// (0 inside), a column with fmaf(D1, D1, RN(D0^2)) > g2 is ineligible for every lane.  The surviving columns (the ballot) are
// then gated exactly per lane, one column at a time; TMEM is read only for a column
// some lane passes.  Returns false (nothing done) when too many columns survive for
// the per-column loop to beat the packed filter; the caller then runs epi_chunk.
constexpr int kSparseMaxCols = 10;

template <int KT, int JP>
__device__ __forceinline__ bool epi_chunk_sorted(uint32_t taddr, int64_t jbase, int nvalid,
                                                 const float* __restrict__ inv_sm, const float* __restrict__ jsm,
                                                 const float (&qj)[JP], float iq, float g2, float bound, int k,
                                                 float wlo, float whi, float wlo1, float whi1, int lane,
                                                 TopK<KT, int32_t>& top) {
  const float p0 = jsm[lane], p1 = jsm[kBlockN + lane];
  const float d0 = p0 < wlo ? __fsub_rn(wlo, p0) : (p0 > whi ? __fsub_rn(whi, p0) : 0.0f);
  const float d1 = p1 < wlo1 ? __fsub_rn(wlo1, p1) : (p1 > whi1 ? __fsub_rn(whi1, p1) : 0.0f);
  uint32_t m = __ballot_sync(0xffffffffu, __fmaf_rn(d1, d1, __fmul_rn(d0, d0)) <= g2);
  if (__popc(m) > kSparseMaxCols) return false;
  while (m != 0u) {
    const int c = __ffs(m) - 1;
    m &= m - 1u;
    float ds = 0.0f;
    bool ok = true;
#pragma unroll
    for (int g = 0; g < JP / 4; ++g) {
      if (!__any_sync(0xffffffffu, ok)) break;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float df = __fsub_rn(qj[4 * g + u], jsm[(4 * g + u) * kBlockN + c]);
        ds = __fmaf_rn(df, df, ds);
      }
      ok = ok && (ds <= g2);
    }
    if (!__any_sync(0xffffffffu, ok)) continue;
    const uint32_t v = ptx::tmem_ld1(taddr + (uint32_t)c);
    ptx::tmem_wait_ld();
    const float s = __fmul_rn(__fmul_rn(__uint_as_float(v), iq), inv_sm[c]);
    if (ok && s > top.kth_s && s >= bound && c < nvalid) top.insert_monotone(s, (int32_t)(jbase + c), k);
  }
  return true;
}

// 168 registers is the ceiling for 10 warps per CTA: warps are spread over the 4 SM
// sub-partitions (3 + 3 + 2 + 2) and each holds 16 K registers, so 3 x 32 x 168 = 16128
// fits while 176 fails at launch ("too many resources").  KT = 64 spills a little.
template <int KT, int JP, int CG, int CL>
__global__ void __maxnreg__(168)
    match_tc_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_pool,
                    const TcParams prm) {
  constexpr int STAGES = stages_for<JP, CG>();
  constexpr uint32_t AUXJ = Aux<JP>::j_bytes;
  constexpr uint32_t AUX = Aux<JP>::bytes;
  constexpr uint32_t BBYTES = Geo<CG>::b_bytes;
  constexpr uint32_t STAGE = Geo<CG>::stage_bytes;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // keep every pointer derived from smem_raw so loads stay in the shared window
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                   // STAGES x 16 KB
  uint8_t* sB = smem + STAGES * kABytes;                // STAGES x BBYTES
  uint8_t* sAux = smem + STAGES * STAGE;                // kAuxDepth x AUX
  uint64_t* bars = reinterpret_cast<uint64_t*>(sAux + kAuxDepth * AUX);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* afull = tfull + 4;
  uint64_t* aempty = afull + kAuxDepth;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(aempty + kAuxDepth);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // CL = CTAs per cluster: CG (one tile per cluster), or 2 * CG = two CTA pairs that
  // work on the same pool rows with different query tiles, each CTA loading half of its
  // pool rows and multicasting them to its counterpart in the other pair (the pool
  // operand's L2 -> SM traffic halves)
  constexpr int NPAIR = CL / CG;
  const uint32_t crank = CL > 1 ? ptx::cluster_ctarank() : 0u;
  const uint32_t pair = crank / CG, prank = crank % CG;   // pair in the cluster, rank in the pair
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int n_qg = prm.n_qt / NPAIR;                      // query-tile groups (one per unit)

  constexpr int kProducerWarp = 4 * kEpiHalves, kMmaWarp = 4 * kEpiHalves + 1;
  if (warp == kProducerWarp && lane == 0) {
    ptx::prefetch_tmap(&tmap_q);
    ptx::prefetch_tmap(&tmap_pool);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], NPAIR);   // one MMA commit per pair whose loads land here
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 4 * kEpiHalves * CG);
    }
    for (int i = 0; i < kAuxDepth; ++i) {
      ptx::mbar_init(&afull[i], 1);
      ptx::mbar_init(&aempty[i], 4 * kEpiHalves);
    }
    ptx::fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    ptx::tmem_alloc<CG>(tmem_holder, kTmemCols);
    ptx::tmem_relinquish<CG>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (CL > 1) ptx::cluster_sync();   // peer barriers initialised before any remote traffic
  ptx::tc_fence_after();
  // launched as a programmatic dependent of the query prep: everything above (barrier
  // init, TMEM allocation, descriptor prefetch) overlapped it; its outputs (staged
  // queries, norms, joints, zeroed bounds / slots) are read only below
  ptx::griddep_wait();
  const uint32_t tmem_base = *tmem_holder;

  const int n_kb = prm.d / kBlockK;

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ TMA producer
    // Whole warp walks the loop and waits (uniform control flow), one elected lane issues.
    {
      const uint32_t full_leader0 = CG == 2 ? ptx::mapa(ptx::smem_u32(&full[0]), pair * CG) : 0u;
      const uint16_t mc_mask = (uint16_t)((1u << crank) | (1u << (crank ^ (uint32_t)CG)));   // NPAIR == 2
      const uint64_t pol_q = ptx::policy_evict_last();
      const uint64_t pol_pool = prm.n_qt > 1 ? ptx::policy_evict_normal() : ptx::policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      uint32_t tile_count = 0;
      uint32_t wave = 0;
      for (int u = cid; u < prm.n_units; u += ncl, ++wave) {
        const int sp = u / n_qg, qt = (u % n_qg) * NPAIR + (int)pair;
        int t_lo, t_hi;
        split_tiles(sp, prm.S, prm.n_pt, t_lo, t_hi);
        const int qrow0 = qt * kBlockM * CG + (int)prank * kBlockM;
        // Wave lockstep: the units sharing a row split run in the same wave (split-major
        // order) and re-read its rows from L2 only while they stay within ~1 ms of each
        // other.  Static striding lets per-unit jitter accumulate across waves (measured
        // on C4: 4 ms start spread, 13x DRAM re-reads), so no producer starts wave w
        // before every CTA has issued all loads of wave w-1.  Best effort: the wait is
        // bounded (~10 ms), so a grid that is not fully co-resident (MPS, concurrent
        // kernels) still progresses -- the lockstep only ever affects speed, never results.
        if (wave > 0) {
          const uint32_t need = wave * gridDim.x;
          for (int it = 0; it < (1 << 16) && *reinterpret_cast<volatile uint32_t*>(prm.wave_ctr) < need; ++it)
            __nanosleep(128);
          __syncwarp();   // lanes may leave the spin at different iterations
        }
        for (int t = t_lo; t < t_hi; ++t, ++tile_count) {
          const int abuf = (int)(tile_count % kAuxDepth);
          const uint32_t ause = tile_count / kAuxDepth;
          ptx::mbar_wait(&aempty[abuf], (ause & 1u) ^ 1u);
          if (ptx::elect_one()) {
            uint8_t* aux = sAux + abuf * AUX;
            ptx::mbar_arrive_expect_tx(&afull[abuf], AUX);
            ptx::bulk_load(aux, prm.pool_joints + (int64_t)t * kBlockN * JP, AUXJ, &afull[abuf]);
            ptx::bulk_load(aux + AUXJ, prm.pool_inv + (int64_t)t * kBlockN, kBlockN * 4, &afull[abuf]);
          }
          __syncwarp();
          const int prow0 = t * kBlockN + (int)prank * (int)Geo<CG>::b_rows;
          for (int kb = 0; kb < n_kb; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1u);
            if (ptx::elect_one()) {
              constexpr bool load_a = true, load_b = true;
              constexpr uint32_t bytes = STAGE;
              if (CG == 1) {
                ptx::mbar_arrive_expect_tx(&full[stage], bytes);
                if (load_a) ptx::tma_load_2d(sA + stage * kABytes, &tmap_q, &full[stage], kb * kBlockK, qrow0, pol_q);
                if (load_b)
                  ptx::tma_load_2d(sB + stage * BBYTES, &tmap_pool, &full[stage], kb * kBlockK, prow0, pol_pool);
              } else {
                if (prank == 0) ptx::mbar_arrive_expect_tx(&full[stage], CG * bytes);
                const uint32_t fb = full_leader0 + (uint32_t)(stage * sizeof(uint64_t));
                if (load_a) ptx::tma_load_2d_pair(sA + stage * kABytes, &tmap_q, fb, kb * kBlockK, qrow0, pol_q);
                if (NPAIR == 1) {
                  if (load_b)
                    ptx::tma_load_2d_pair(sB + stage * BBYTES, &tmap_pool, fb, kb * kBlockK, prow0, pol_pool);
                } else if (load_b) {
                  // half of this CTA's pool rows, into both pairs (same CTA-relative offset);
                  // completion goes to each destination pair's leader barrier
                  constexpr uint32_t half = BBYTES / 2;
                  ptx::tma_load_2d_pair_mc(sB + stage * BBYTES + pair * half, &tmap_pool, &full[stage], mc_mask,
                                           kb * kBlockK, prow0 + (int)pair * (int)(Geo<CG>::b_rows / 2), pol_pool);
                }
              }
            }
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
        if (ptx::elect_one()) atomicAdd(prm.wave_ctr, 1u);
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (leader)
    // The whole warp walks the (uniform) loop and waits; one elected lane issues.  The
    // smem descriptors of a stage are the base descriptors plus the stage offset (the
    // 14-bit start-address field never carries: smem < 256 KB), so an UMMA costs a few
    // uniform integer ops instead of a per-issue descriptor rebuild.
    if (prank == 0) {
      // commits: stage release to every CTA whose shared memory the stage's loads filled
      // (this pair, plus the other pair's when the pool rows are multicast); accumulator
      // ready to this pair only
      const uint16_t empty_mask = (uint16_t)(NPAIR == 1 ? 0x3u : 0xFu);
      const uint16_t tfull_mask = (uint16_t)(0x3u << (pair * CG));
      int stage = 0;
      uint32_t phase = 0;
      uint32_t tile_count = 0;
      const uint64_t da0 = ptx::sdesc_k_sw128(ptx::smem_u32(sA));
      const uint64_t db0 = ptx::sdesc_k_sw128(ptx::smem_u32(sB));
      for (int u = cid; u < prm.n_units; u += ncl) {
        const int sp = u / n_qg;
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
            if (ptx::elect_one()) {
              const uint64_t da = da0 + (uint64_t)((uint32_t)stage * (kABytes >> 4));
              const uint64_t db = db0 + (uint64_t)((uint32_t)stage * (BBYTES >> 4));
#pragma unroll
              for (int kk = 0; kk < kBlockK / 16; ++kk)
                ptx::umma_f16<CG>(d_tmem, da + (uint64_t)(2 * kk), db + (uint64_t)(2 * kk), Geo<CG>::idesc,
                                  (kb | kk) != 0 ? 1u : 0u);
              if (CG == 1)
                ptx::umma_commit<CG>(&empty[stage]);
              else
                ptx::umma_commit_mc(&empty[stage], empty_mask);
            }
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
          if (ptx::elect_one()) {
            if (CG == 1)
              ptx::umma_commit<CG>(&tfull[buf]);
            else
              ptx::umma_commit_mc(&tfull[buf], tfull_mask);
          }
          __syncwarp();
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int lg = warp & 3;           // TMEM lane group accessible to this warp
    const int h = warp >> 2;           // column half
    uint32_t tile_count = 0;
    const bool gated = prm.gated != 0;
    const uint32_t tempty_leader0 = CG == 2 ? ptx::mapa(ptx::smem_u32(&tempty[0]), pair * CG) : 0u;
    for (int u = cid; u < prm.n_units; u += ncl) {
      const int sp = u / n_qg, qt = (u % n_qg) * NPAIR + (int)pair;
      int t_lo, t_hi;
      split_tiles(sp, prm.S, prm.n_pt, t_lo, t_hi);
      const int64_t row_end = min((int64_t)t_hi * kBlockN, prm.L);
      const int qrow = qt * kBlockM * CG + (int)prank * kBlockM + lg * 32 + lane;
      const bool active = qrow < prm.nq;
      float qj[JP];
#pragma unroll
      for (int t = 0; t < JP; ++t) qj[t] = active ? prm.q_joints[(int64_t)qrow * JP + t] : 0.0f;
      uint64_t QQ[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) QQ[t] = ptx::pack2(qj[t], qj[t]);   // JP >= 4
      const float iq = active ? prm.inv_q[qrow] : 0.0f;
      // joint-0 / joint-1 intervals of the warp's active queries (empty warp: no column passes)
      float wlo = active ? qj[0] : CUDART_INF_F, whi = active ? qj[0] : -CUDART_INF_F;
      float wlo1 = active ? qj[1] : CUDART_INF_F, whi1 = active ? qj[1] : -CUDART_INF_F;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        wlo = fminf(wlo, __shfl_xor_sync(0xffffffffu, wlo, o));
        whi = fmaxf(whi, __shfl_xor_sync(0xffffffffu, whi, o));
        wlo1 = fminf(wlo1, __shfl_xor_sync(0xffffffffu, wlo1, o));
        whi1 = fmaxf(whi1, __shfl_xor_sync(0xffffffffu, whi1, o));
      }
      const bool sparse = gated && prm.sorted != 0;
      // the caller's query index: partial lists, the bound and its slots are indexed by it
      const int64_t qout = (active && prm.perm != nullptr) ? (int64_t)prm.perm[qrow] : (int64_t)qrow;
      uint32_t* bnd = prm.bound + (active ? qout : 0);
      float bound = -CUDART_INF_F;
      if (active) {
        const uint32_t b = ptx::ld_relaxed_gpu(bnd);
        if (b) bound = ptx::ord2f(b);
      }
      TopK<KT, int32_t> top;
      top.init(active);
      for (int t = t_lo; t < t_hi; ++t, ++tile_count) {
        const int buf = tile_count & 1;
        const uint32_t use = tile_count >> 1;
        const int abuf = (int)(tile_count % kAuxDepth);
        ptx::mbar_wait(&afull[abuf], (tile_count / kAuxDepth) & 1u);
        ptx::mbar_wait(&tfull[buf], use & 1u);
        ptx::tc_fence_after();
        const uint8_t* aux = sAux + abuf * AUX;
        const float* joints_sm = reinterpret_cast<const float*>(aux);
        const float* inv_sm = reinterpret_cast<const float*>(aux + AUXJ);
        float ie_min = 0.0f, ie_max = 0.0f;   // inverse-norm range of this warp's column half
        if (!gated) {
          const float4 a = lds4(inv_sm + h * kColsPerHalf + 4 * lane);
          ie_min = fminf(fminf(a.x, a.y), fminf(a.z, a.w));
          ie_max = ptx::fmax3(a.x, a.y, fmaxf(a.z, a.w));
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            ie_min = fminf(ie_min, __shfl_xor_sync(0xffffffffu, ie_min, o));
            ie_max = fmaxf(ie_max, __shfl_xor_sync(0xffffffffu, ie_max, o));
          }
        }
#pragma unroll 1
        for (int ch = 0; ch < kColsPerHalf / kChunk; ++ch) {
          const int col0 = h * kColsPerHalf + ch * kChunk;
          const uint32_t taddr = tmem_base + ((uint32_t)(lg * 32) << 16) + (uint32_t)(buf * kBlockN + col0);
          const int64_t jbase = (int64_t)t * kBlockN + col0;
          const int nvalid = (int)max((int64_t)0, min((int64_t)kChunk, row_end - jbase));
          if (sparse && epi_chunk_sorted<KT, JP>(taddr, jbase, nvalid, inv_sm + col0, joints_sm + col0, qj, iq,
                                                 prm.g2, bound, prm.k, wlo, whi, wlo1, whi1, lane, top))
            continue;
          if (gated)
            epi_chunk<KT, JP, true>(taddr, jbase, nvalid, inv_sm + col0, joints_sm + col0, QQ, qj, iq, ie_min, ie_max,
                                    prm.g2, bound, prm.k, top);
          else
            epi_chunk<KT, JP, false>(taddr, jbase, nvalid, inv_sm + col0, joints_sm + col0, QQ, qj, iq, ie_min, ie_max,
                                     prm.g2, bound, prm.k, top);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 1)
            ptx::mbar_arrive(&tempty[buf]);
          else
            ptx::mbar_arrive_cluster(tempty_leader0 + (uint32_t)(buf * sizeof(uint64_t)));
          ptx::mbar_arrive(&aempty[abuf]);
        }
        // share the admission bound with the other splits of this query
        // Geometric schedule (after 1, 2, 4, 8, ... tiles of the unit, and at its end):
        // bounds move fast early and slowly later, and the reload is an L2 round trip
        // whose latency the two epilogue warps of a sub-partition cannot hide when the
        // MMA of a tile is short (d = 768: the per-tile refresh left the tensor pipe
        // idle ~20 % of the time).
        const int done = t - t_lo + 1;
        if ((done & (done - 1)) == 0 || t + 1 == t_hi) {
          if (active) {
            if (top.kth_s > -CUDART_INF_F) atomicMax(bnd, ptx::f2ord(top.kth_s));
            const uint32_t b = ptx::ld_relaxed_gpu(bnd);
            if (b) bound = fmaxf(bound, ptx::ord2f(b));
            if (prm.slots != nullptr) {
              // union bound: list l keeps its best score in slot l mod k; slots hold
              // rows of disjoint list groups, so with all k slots filled their minimum
              // is the score of one of k distinct rows, <= the k-th best of the pool
              uint32_t* sl = prm.slots + qout * KT;
              if (top.s[0] > -CUDART_INF_F) atomicMax(sl + (sp * kEpiHalves + h) % prm.k, ptx::f2ord(top.s[0]));
              uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
              for (int r = 0; r < KT; r += 4) {
                const uint4 v = __ldcg(reinterpret_cast<const uint4*>(sl + r));
                mn = min(mn, min(min(r < prm.k ? v.x : ~0u, r + 1 < prm.k ? v.y : ~0u),
                                 min(r + 2 < prm.k ? v.z : ~0u, r + 3 < prm.k ? v.w : ~0u)));
              }
              if (mn != 0u) bound = fmaxf(bound, ptx::ord2f(mn));
            }
          }
        }
      }
      if (active) {
        const int64_t base = (qout * prm.P + (int64_t)sp * kEpiHalves + h) * KT;
#pragma unroll
        for (int r = 0; r < KT; r += 4) {
          *reinterpret_cast<float4*>(prm.part_s + base + r) =
              make_float4(top.s[r], top.s[r + 1], top.s[r + 2], top.s[r + 3]);
          *reinterpret_cast<int4*>(prm.part_i + base + r) = make_int4(top.i[r], top.i[r + 1], top.i[r + 2], top.i[r + 3]);
        }
      }
    }
  }

  ptx::griddep_launch_dependents();   // the merge may be scheduled (it waits for our completion)
  ptx::tc_fence_before();
  __syncthreads();
  if (CL > 1) ptx::cluster_sync();   // no CTA leaves while a peer may still signal it
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, kTmemCols);
  }
}

template <int KT, int JP, int CG, int CL>
cudaError_t launch_tc_t(Pool& p, const TcParams& prm, int grid, cudaStream_t s) {
  auto kern = match_tc_kernel<KT, JP, CG, CL>;
  const size_t smem = smem_for<JP, CG>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreadsTc);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see griddep_wait()
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, p.tmap_q, CG == 1 ? p.tmap_pool : CL == CG ? p.tmap_pool2 : p.tmap_pool4,
                            prm);
}

template <int KT, int CG, int CL>
cudaError_t launch_tc_kt(Pool& p, const TcParams& prm, int grid, cudaStream_t s) {
  switch (p.JP) {
    case 4: return launch_tc_t<KT, 4, CG, CL>(p, prm, grid, s);
    case 8: return launch_tc_t<KT, 8, CG, CL>(p, prm, grid, s);
    default: return launch_tc_t<KT, 16, CG, CL>(p, prm, grid, s);
  }
}

template <int CG, int CL>
cudaError_t launch_tc_cg(Pool& p, const MatchArgs& a, const TcParams& prm, int grid, cudaStream_t s) {
  switch (a.KT) {
    case 8: return launch_tc_kt<8, CG, CL>(p, prm, grid, s);
    case 16: return launch_tc_kt<16, CG, CL>(p, prm, grid, s);
    case 32: return launch_tc_kt<32, CG, CL>(p, prm, grid, s);
    default: return launch_tc_kt<64, CG, CL>(p, prm, grid, s);
  }
}

}  // namespace

int tc_query_tile(int cg) { return kBlockM * cg; }

// Clusters of `cl` CTAs of the CTA-pair kernel that can be co-resident (clusters must fit
// within a GPC, so this can be below num_sms / cl).  0 on error.
int tc_max_active_clusters(int cl) {
  auto kern = cl == 4 ? match_tc_kernel<16, 16, 2, 4> : match_tc_kernel<16, 16, 2, 2>;
  const size_t smem = smem_for<16, 2>();
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(cl * 64));
  cfg.blockDim = dim3(kThreadsTc);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void*)kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

cudaError_t launch_match_tc(Pool& p, const MatchArgs& a, int32_t S, int32_t grid, int32_t cg, int32_t cl,
                            bool sorted, cudaStream_t s) {
  TcParams prm{};
  prm.inv_q = p.q_inv;
  prm.q_joints = p.q_joints;
  prm.pool_inv = p.inv_norm;
  prm.pool_joints = p.joints;
  prm.part_s = p.part_s;
  prm.part_i = p.part_i;
  prm.bound = p.bound;
  prm.wave_ctr = p.bound + a.nq;
  prm.perm = sorted ? p.q_perm : nullptr;
  prm.sorted = sorted ? 1 : 0;
  prm.L = p.local;
  prm.nq = a.nq;
  prm.d = p.cfg.dim;
  prm.n_qt = (a.nq + kBlockM * cg - 1) / (kBlockM * cg);
  prm.n_pt = (int32_t)((p.local + kBlockN - 1) / kBlockN);
  prm.S = S;
  prm.n_units = prm.n_qt / (cl / cg) * S;   // units = (query-tile group, row split)
  prm.k = a.k;
  prm.gated = a.gated;
  prm.P = S * kEpiHalves;
  prm.g2 = a.g2;
  cudaError_t e = cudaSuccess;
  if (!a.zeroed && (e = cudaMemsetAsync(p.bound, 0, (size_t)(a.nq + 1) * sizeof(uint32_t), s)) != cudaSuccess)
    return e;
  // ungated: the union bound needs >= k lists per query (each list fills one slot)
  prm.slots = (!a.gated && prm.P >= a.k) ? p.slots : nullptr;   // a.slots says so to the merge
  if (prm.slots != nullptr && !a.zeroed) {
    e = cudaMemsetAsync(p.slots, 0, (size_t)prm.n_qt * kBlockM * cg * a.KT * sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
  }
  if (cl != cg && (cg != 2 || cl != 4 || prm.n_qt % 2 != 0)) return cudaErrorInvalidValue;
  e = cg == 1 ? launch_tc_cg<1, 1>(p, a, prm, grid, s)
              : cl == 2 ? launch_tc_cg<2, 2>(p, a, prm, grid, s) : launch_tc_cg<2, 4>(p, a, prm, grid, s);
  ++p.launches;
  return e;
}

}  // namespace ams

