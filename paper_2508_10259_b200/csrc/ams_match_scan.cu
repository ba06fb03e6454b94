// ams_match_scan.cu -- small-batch tcgen05 matcher (nq <= 128): pool rows on the MMA M
// side, queries on N.
//
// Same method as ams_match_tc.cu (3.2.1 "comparing the similarity";
// north_star metric, gate, top-k, tie rule):
//   acc(i,j)  = sum_t q_it * e_jt          bf16 x bf16 -> fp32 on the tensor cores
//   s(i,j)    = (acc * inv_q_i) * inv_e_j  fp32
//   gate(i,j) = canonical fp32 sum_t (r_it - p_jt)^2 <= g2
//   top-k by (s desc, j asc) per query.
//
// Why a second kernel.  A batch of nq <= 128 queries is HBM-bound (one pool row is
// 2d bytes for 2*nq*d flop).  In match_tc_kernel the queries are the MMA M side, which
// is 128 rows whatever nq is: a 1-query lookup does 128x the tensor work it needs.  On a
// long scan at the 1 kW cap that wasted work is what sets the clock (C5 streaming: SM
// clock 611-645 MHz median, and at that clock an M = 128 scan of d = 4096 rows is
// tensor-bound, not HBM-bound).  Here the pool tile is the M side (two M = 128 MMAs per
// 256-row tile) and the queries are N = round_up(nq, 32): the tensor work follows nq.
//
// Tiling: a tile is 256 pool rows (two 128-row MMA halves) x NQ queries, K advances 64
// bf16 per pipeline stage (one 128-B swizzle atom).  TMEM: two accumulator buffers of
// 2*NQ columns; half h of buffer b at columns b*2NQ + h*NQ, lane = pool row (mod 128).
//
// CTA pairs (129-256 queries) can run "wide" (W = 2, opt-in): a pipeline stage carries the pair's
// 128-row halves of TWO consecutive tiles per CTA (two cta_group::2 MMAs, M = 256 each)
// against one stage of N/2 query rows per CTA, so every query byte staged from L2 serves
// 512 pool rows instead of 256.  The L2 -> SM operand traffic of a call drops from
// pool x (1 + N/256) to pool x (1 + N/512) -- at N = 224 from 1.88x to 1.44x the pool --
// which is what bounded the narrow pair (LTS throughput, ~9.5 TB/s at the capped clock).
// The price is TMEM: 2 halves x N columns fill it, so the accumulator is single-
// buffered; the TMA ring keeps streaming the next super-tile while the epilogue drains.
//
// Warp roles (192 threads, 1 CTA/SM): warps 0..3 epilogue (warp w reads TMEM lanes
// 32w.. = pool rows 32w+lane and 128+32w+lane of each tile), warp 4 TMA producer
// (pool + query tiles into a STAGES ring, per-tile joints/inv_norm into a 2-deep aux
// ring), warp 5 TMEM allocator + tcgen05.mma issuer.
//
// Epilogue, per warp, half tile (32 rows) and 32-query slot: one tcgen05.ld.x32 gives
// lane r the raw scores of row r against the slot's 32 queries.  Lanes are rows here,
// but the running top-k lists are per query, so each warp keeps them in registers
// with lane q owning query (slot*32 + q) -- the same register TopK as match_tc_kernel.
// A row-side filter decides whether the block can touch any list: gated, the
// canonical partial distance over joints 0..3 (a lower bound of the full sum: RN is
// monotone and every term >= 0), then the exact canonical gate for the pairs that
// pass; ungated, the exact score against the query's threshold (mirrored in shared
// memory as max(KT-th best, shared bound)).  Only then is the 32x32 block of scores
// (-inf where ineligible) transposed through shared memory (padded rows: conflict-
// free) so lane q scans its query's 32 rows in increasing row order and inserts with
// TopK::insert_monotone.  Lists are per (query, split, warp) and go to the same
// [nq][P][KT] partial layout merge_partials_kernel merges; the per-query bound in
// global memory is shared across CTAs exactly as in match_tc_kernel (a list's KT-th
// best is <= the global k-th best, so s < bound can never enter; s == bound is kept
// for the index tie rule), refreshed on a geometric tile schedule.
#include <cuda_bf16.h>
#include <math_constants.h>

#include "ams_internal.cuh"
#include "ams_ptx.cuh"
#include "ams_topk.cuh"

namespace ams {
namespace {

constexpr int kScanEpiWarps = 4;
constexpr int kScanThreads = 32 * (kScanEpiWarps + 2);   // 192
constexpr uint32_t kScanABytes = kBlockN * kBlockK * 2;  // 32 KB: 256 pool rows x 128 B
constexpr uint32_t kScanHalfBytes = kScanABytes / 2;     // 128 rows: the second MMA half
constexpr int kScanListRegs = 2048;                      // max (32-query slots) x KT per lane
constexpr size_t kSmemLimit = 232448;                    // max dynamic smem per CTA (227 KB)
constexpr int kTPad = 33;                                // transpose row stride (floats)

struct ScanParams {
  const float* inv_q;        // [q_pad]
  const float* q_joints;     // [q_pad, JP]
  const float* pool_inv;     // [cap_pad]
  const float* pool_joints;  // [cap_pad/256][JP][256]
  float* part_s;             // [nq][P][KT]
  int32_t* part_i;
  uint32_t* bound;           // [nq] ordered-u32 admission lower bound (0 = none)
  uint32_t* slots;           // [nq][KT] union-bound slots (ordered-u32; ungated with P >= k, else null)
  float* glist_s;            // CG = 2: per (CTA, epilogue warp) lists [slot][KT][32 lanes]
  int32_t* glist_i;
  int64_t L;                 // local rows
  int32_t nq, NQ, NM, d, n_pt, S, P, stages, k;   // NQ = round_up(nq, 32): epilogue slots / TMEM
                                                  // layout; NM = round_up(nq, 16): the MMA's N
  uint32_t b_bytes;          // query stage bytes (box rows x 128 B)
  uint32_t idesc;            // kind::f16, M = 128, N = NQ
  float g2;
};

// shared-memory layout (byte offsets from the 1024-aligned base), host and device
struct ScanLayout {
  uint32_t a, b, aux, tr, qj, iq, thr, em, ls, li, bars, total;
};

// cg = 2: a CTA stages 128 of the pair's 256 pool rows per stage
__host__ __device__ inline ScanLayout scan_layout(int stages, uint32_t b_bytes, int JP, int NQ, int cg, int KT,
                                                  int W) {
  ScanLayout l{};
  const uint32_t rows = (uint32_t)(kBlockN / cg * W);   // pool rows per CTA and stage
  uint32_t o = 0;
  l.a = o;
  o += (uint32_t)stages * rows * kBlockK * 2;
  l.b = o;
  o += (uint32_t)stages * b_bytes;
  l.aux = o;
  o += 2u * (rows * JP * 4 + rows * 4);   // joints + inv of this CTA's rows
  l.tr = o;
  o += (uint32_t)(kScanEpiWarps * 32 * kTPad * 4 + 64);   // + keep 16-B alignment below
  l.qj = o;
  o += (uint32_t)(JP * NQ * 4);
  l.iq = o;
  o += (uint32_t)(NQ * 4);
  l.thr = o;
  o += (uint32_t)(kScanEpiWarps * NQ * 4);
  l.em = o;   // gate masks [warps][halves][NQ / 32 slots][32 lanes]
  o += (uint32_t)(kScanEpiWarps * (cg == 1 ? 2 : W) * NQ * 4);
  l.ls = l.li = o;   // (lists: registers for cg = 1, global memory for cg = 2)
  l.bars = o;
  o += 256;
  l.total = o + 1024;   // alignment slack
  return l;
}

// split sp of S over the pool's tiles, in whole super-tiles of W tiles (the last may be
// short: its missing tiles are past the pool and load / score nothing)
__device__ __forceinline__ void scan_split(int sp, int S, int n_pt, int W, int& t_lo, int& t_hi) {
  const int n_st = (n_pt + W - 1) / W;
  t_lo = W * (int)((int64_t)sp * n_st / S);
  t_hi = min(n_pt, W * (int)((int64_t)(sp + 1) * n_st / S));
}

// CG = 1: one CTA per 256-row tile (two M = 128 MMAs), nq <= 128.  CG = 2: a CTA pair
// per 256-row tile (one tcgen05.mma.cta_group::2 with M = 256: each CTA stages 128 pool
// rows and half of the N query rows), 128 < nq <= 256; each CTA's epilogue owns its 128
// rows against all N queries.
template <int KT, int JP, bool GATED, int CG, int W>
__global__ void __launch_bounds__(kScanThreads, 1)
    match_scan_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_pool,
                      const ScanParams prm) {
  // CG = 2 keeps the lists in global memory (L2-resident, private to each warp, touched
  // only on inserts): in registers 8 slots (112 registers) made ptxas serialise the gate
  // filter's loads and spill; in shared memory they cost pipeline stages (C5: 3 stages,
  // 7.4 ms vs 6.3 ms per 129-256-query call)
  constexpr bool SMEM_LISTS = CG == 2;   // (name kept: the lists are out of registers)
  static_assert(W == 1 || CG == 2, "wide stages are a CTA-pair mode");
  constexpr int HALVES = CG == 1 ? 2 : W;          // 128-row MMA halves per CTA and stage
  constexpr int NBUF = W == 1 ? 2 : 1;             // TMEM accumulator buffers (2 * HALVES * NQ <= 512)
  constexpr int AROWS = 128 * HALVES;              // super-tile rows this CTA owns (aux ring)
  constexpr uint32_t AUXJ = AROWS * JP * 4;
  constexpr uint32_t AUX = AUXJ + AROWS * 4;
  constexpr uint32_t ABYTES = kScanHalfBytes * HALVES;   // pool rows staged per CTA and stage
  constexpr int NQMAX = 128 * CG;
  constexpr int NSL0 = kScanListRegs / (32 * KT);
  constexpr int NSL = NSL0 < NQMAX / 32 ? NSL0 : NQMAX / 32;   // 32-query slots per lane
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int NQ = prm.NQ;
  const int STAGES = prm.stages;
  const ScanLayout lay = scan_layout(STAGES, prm.b_bytes, JP, NQ, CG, KT, W);
  uint8_t* sA = smem + lay.a;
  uint8_t* sB = smem + lay.b;
  uint8_t* sAux = smem + lay.aux;
  float* trs = reinterpret_cast<float*>(smem + lay.tr);   // [warps][32][kTPad]
  float* qjs = reinterpret_cast<float*>(smem + lay.qj);   // [JP][NQ]
  float* iqs = reinterpret_cast<float*>(smem + lay.iq);   // [NQ]
  float* thr = reinterpret_cast<float*>(smem + lay.thr);  // [warps][NQ]
  uint32_t* ems = reinterpret_cast<uint32_t*>(smem + lay.em);   // [warps][HALVES][NQ/32][32]
  float* lsm = prm.glist_s + (int64_t)blockIdx.x * kScanEpiWarps * NSL * KT * 32;   // SMEM_LISTS
  int32_t* lim = prm.glist_i + (int64_t)blockIdx.x * kScanEpiWarps * NSL * KT * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.bars);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* afull = tfull + 4;
  uint64_t* aempty = tfull + 6;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tfull + 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = CG == 2 ? ptx::cluster_ctarank() : 0u;
  const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;
  constexpr int kProducerWarp = kScanEpiWarps, kMmaWarp = kScanEpiWarps + 1;
  if (warp == kProducerWarp && lane == 0) {
    ptx::prefetch_tmap(&tmap_q);
    ptx::prefetch_tmap(&tmap_pool);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kScanEpiWarps * CG);
      ptx::mbar_init(&afull[i], 1);
      ptx::mbar_init(&aempty[i], kScanEpiWarps);
    }
    ptx::fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    ptx::tmem_alloc<CG>(tmem_holder, 512);
    ptx::tmem_relinquish<CG>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (CG == 2) ptx::cluster_sync();   // peer barriers initialised before any remote traffic
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // launched as a programmatic dependent of the query prep: everything above (barrier
  // init, TMEM allocation, descriptor prefetch) overlapped it; its outputs (staged
  // queries, norms, joints, zeroed bounds / slots) are read only below
  ptx::griddep_wait();
  const int n_kb = prm.d / kBlockK;

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ TMA producer
    const uint64_t pol_q = ptx::policy_evict_last();
    const uint64_t pol_pool = ptx::policy_evict_first();   // every pool byte is read once
    const uint32_t tx = ABYTES + prm.b_bytes;
    const uint32_t full_leader0 = CG == 2 ? ptx::mapa(ptx::smem_u32(&full[0]), 0) : 0u;
    const int qrow0 = (int)crank * (prm.NM / CG);   // this CTA's query rows (the B half)
    int stage = 0;
    uint32_t phase = 0, tile_count = 0;
    for (int u = cid; u < prm.S; u += ncl) {
      int t_lo, t_hi;
      scan_split(u, prm.S, prm.n_pt, W, t_lo, t_hi);
      for (int t = t_lo; t < t_hi; t += W, ++tile_count) {
        const int buf = tile_count & 1;
        const uint32_t use = tile_count >> 1;
        ptx::mbar_wait(&aempty[buf], (use & 1u) ^ 1u);
        if (ptx::elect_one()) {
          uint8_t* aux = sAux + buf * AUX;
          if (CG == 1) {
            ptx::mbar_arrive_expect_tx(&afull[buf], AUX);
            ptx::bulk_load(aux, prm.pool_joints + (int64_t)t * kBlockN * JP, AUXJ, &afull[buf]);
            ptx::bulk_load(aux + AUXJ, prm.pool_inv + (int64_t)t * kBlockN, AROWS * 4, &afull[buf]);
          } else {   // this CTA's 128 columns of each joint row of the [JP][256] block of tile t + h
            const int hv = min(W, prm.n_pt - t);   // a super-tile past the last tile loads nothing for it
            ptx::mbar_arrive_expect_tx(&afull[buf], (uint32_t)hv * 128u * (JP + 1) * 4u);
            for (int h = 0; h < hv; ++h) {
#pragma unroll
              for (int tj = 0; tj < JP; ++tj)
                ptx::bulk_load(aux + (tj * AROWS + h * 128) * 4,
                               prm.pool_joints + ((int64_t)(t + h) * JP + tj) * kBlockN + crank * 128, 128 * 4,
                               &afull[buf]);
              ptx::bulk_load(aux + AUXJ + h * 128 * 4, prm.pool_inv + (int64_t)(t + h) * kBlockN + crank * 128, 128 * 4,
                             &afull[buf]);
            }
          }
        }
        __syncwarp();
        for (int kb = 0; kb < n_kb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1u);
          if (ptx::elect_one()) {
            if (CG == 1) {
              ptx::mbar_arrive_expect_tx(&full[stage], tx);
              ptx::tma_load_2d(sA + stage * ABYTES, &tmap_pool, &full[stage], kb * kBlockK, t * kBlockN, pol_pool);
              ptx::tma_load_2d(sB + stage * prm.b_bytes, &tmap_q, &full[stage], kb * kBlockK, 0, pol_q);
            } else {
              if (crank == 0) ptx::mbar_arrive_expect_tx(&full[stage], CG * tx);
              const uint32_t fb = full_leader0 + (uint32_t)(stage * sizeof(uint64_t));
#pragma unroll
              for (int h = 0; h < W; ++h)   // rows past the pool's storage are zero-filled by the TMA
                ptx::tma_load_2d_pair(sA + stage * ABYTES + h * kScanHalfBytes, &tmap_pool, fb, kb * kBlockK,
                                      (t + h) * kBlockN + (int)crank * 128, pol_pool);
              ptx::tma_load_2d_pair(sB + stage * prm.b_bytes, &tmap_q, fb, kb * kBlockK, qrow0, pol_q);
            }
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (pair leader)
    const uint64_t da0 = ptx::sdesc_k_sw128(ptx::smem_u32(sA));
    const uint64_t db0 = ptx::sdesc_k_sw128(ptx::smem_u32(sB));
    int stage = 0;
    uint32_t phase = 0, tile_count = 0;
    for (int u = cid; u < prm.S && crank == 0; u += ncl) {
      int t_lo, t_hi;
      scan_split(u, prm.S, prm.n_pt, W, t_lo, t_hi);
      for (int t = t_lo; t < t_hi; t += W, ++tile_count) {
        const int buf = NBUF == 2 ? (int)(tile_count & 1) : 0;
        const uint32_t use = NBUF == 2 ? tile_count >> 1 : tile_count;
        ptx::mbar_wait(&tempty[buf], (use & 1u) ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d0 = tmem_base + (uint32_t)(buf * HALVES * NQ);
        for (int kb = 0; kb < n_kb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            const uint64_t da = da0 + (uint64_t)((uint32_t)stage * (ABYTES >> 4));
            const uint64_t db = db0 + (uint64_t)((uint32_t)stage * (prm.b_bytes >> 4));
#pragma unroll
            for (int h = 0; h < HALVES; ++h)
#pragma unroll
              for (int kk = 0; kk < kBlockK / 16; ++kk)
                ptx::umma_f16<CG>(d0 + (uint32_t)(h * NQ), da + (uint64_t)(h * (kScanHalfBytes >> 4) + 2 * kk),
                                  db + (uint64_t)(2 * kk), prm.idesc, (kb | kk) != 0 ? 1u : 0u);
            ptx::umma_commit<CG>(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (ptx::elect_one()) ptx::umma_commit<CG>(&tfull[buf]);
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int lg = warp;   // TMEM lanes 32*lg..: rows 32*lg + lane and 128 + 32*lg + lane
    const int nq = prm.nq;
    const int nsl = NQ / 32;   // 32-query slots in use (<= NSL)
    for (int i = threadIdx.x; i < NQ * JP; i += 32 * kScanEpiWarps) {
      const int c = i / JP, t = i % JP;
      qjs[t * NQ + c] = c < nq ? prm.q_joints[(int64_t)c * JP + t] : 0.0f;
    }
    for (int c = threadIdx.x; c < NQ; c += 32 * kScanEpiWarps) iqs[c] = c < nq ? prm.inv_q[c] : 0.0f;
    ptx::named_bar_sync(1, 32 * kScanEpiWarps);
    float* tr = trs + lg * 32 * kTPad;
    float* mythr = thr + lg * NQ;
    const uint32_t tempty_leader0 = CG == 2 ? ptx::mapa(ptx::smem_u32(&tempty[0]), 0) : 0u;
    uint32_t tile_count = 0;
    for (int u = cid; u < prm.S; u += ncl) {
      int t_lo, t_hi;
      scan_split(u, prm.S, prm.n_pt, W, t_lo, t_hi);
      // lane q owns query sl*32 + q of every slot sl: its list and its shared bound
      TopK<KT, int32_t> top[SMEM_LISTS ? 1 : NSL];
      float kth_s[NSL], best_s[NSL];   // SMEM_LISTS: each list's KT-th and best score
      float* wls = lsm + lg * NSL * KT * 32;   // this warp's lists (SMEM_LISTS)
      int32_t* wli = lim + lg * NSL * KT * 32;
      float bnd[NSL];
#pragma unroll
      for (int sl = 0; sl < NSL; ++sl) {
        const int c = sl * 32 + lane;
        const bool act = sl < nsl && c < nq;
        if constexpr (SMEM_LISTS) {
          kth_s[sl] = act ? -CUDART_INF_F : CUDART_INF_F;   // inactive: never admits
          best_s[sl] = -CUDART_INF_F;
          if (sl < nsl)
#pragma unroll
            for (int rr = 0; rr < KT; ++rr) {
              wls[(sl * KT + rr) * 32 + lane] = -CUDART_INF_F;
              wli[(sl * KT + rr) * 32 + lane] = -1;
            }
        } else {
          top[SMEM_LISTS ? 0 : sl].init(act);   // inactive: kth = +inf, never admits
        }
        bnd[sl] = -CUDART_INF_F;
        if (act) {
          const uint32_t v = ptx::ld_relaxed_gpu(prm.bound + c);
          if (v) bnd[sl] = ptx::ord2f(v);
        }
        if (sl < nsl) mythr[c] = act ? bnd[sl] : CUDART_INF_F;
      }
      __syncwarp();
      for (int t = t_lo; t < t_hi; t += W, ++tile_count) {
        const int buf = tile_count & 1;   // aux ring slot
        const uint32_t use = tile_count >> 1;
        const int tb = NBUF == 2 ? buf : 0;   // TMEM accumulator buffer
        const uint32_t tuse = NBUF == 2 ? use : tile_count;
        ptx::mbar_wait(&afull[buf], use & 1u);
        const float* jsm = reinterpret_cast<const float*>(sAux + buf * AUX);
        const float* inv_sm = reinterpret_cast<const float*>(sAux + buf * AUX + AUXJ);
        // Phase A (gated): the joint gate needs no score, so it runs as soon as the tile's
        // joints have landed -- while the MMA is still accumulating the tile -- and leaves
        // per (row half, 32-query slot) masks of the pairs that pass the exact canonical
        // gate.  Phase B holds the accumulators only for blocks with a passing pair (with
        // single-buffered TMEM in the wide pair mode this is what keeps the MMA fed).
        uint32_t* emw = ems + lg * HALVES * NQ;   // this warp's masks, [h][sl][lane]
        if (GATED) {
#pragma unroll 1
          for (int h = 0; h < HALVES; ++h) {
            const int32_t rowbase = CG == 1 ? t * kBlockN + h * 128 + lg * 32
                                            : (t + h) * kBlockN + (int)crank * 128 + lg * 32;
            const bool valid = (int64_t)rowbase + lane < prm.L;
            const int ra = h * 128 + lg * 32 + lane;   // row within this CTA's aux block
            float pj[JP];
#pragma unroll
            for (int tj = 0; tj < JP; ++tj) pj[tj] = jsm[tj * AROWS + ra];
            uint64_t PP[4];
#pragma unroll
            for (int tj = 0; tj < 4; ++tj) PP[tj] = ptx::pack2(pj[tj], pj[tj]);   // JP >= 4
#pragma unroll 1
            for (int sl = 0; sl < nsl; ++sl) {
              const int c0 = sl * 32;
              // partial canonical distance over joints 0..3 for the 32 queries, two at a time
              uint32_t fire = 0;
#pragma unroll
              for (int g = 0; g < 32; g += 4) {
                uint64_t da = 0ull, db = 0ull;
#pragma unroll
                for (int tj = 0; tj < 4; ++tj) {
                  const ulonglong2 q4 = *reinterpret_cast<const ulonglong2*>(qjs + tj * NQ + c0 + g);
                  const uint64_t a = ptx::sub2(q4.x, PP[tj]);
                  da = ptx::fma2(a, a, da);
                  const uint64_t b = ptx::sub2(q4.y, PP[tj]);
                  db = ptx::fma2(b, b, db);
                }
                fire |= (ptx::lo2(da) <= prm.g2 ? 1u : 0u) << g;
                fire |= (ptx::hi2(da) <= prm.g2 ? 1u : 0u) << (g + 1);
                fire |= (ptx::lo2(db) <= prm.g2 ? 1u : 0u) << (g + 2);
                fire |= (ptx::hi2(db) <= prm.g2 ? 1u : 0u) << (g + 3);
              }
              if (!valid) fire = 0u;
              uint32_t elig = 0u;
              if (__reduce_or_sync(0xffffffffu, fire) != 0u) {   // rare: exact canonical gate of the survivors
                while (fire != 0u) {
                  const int c = __ffs(fire) - 1;
                  fire &= fire - 1u;
                  float ds = 0.0f;
#pragma unroll
                  for (int tj = 0; tj < JP; ++tj) {
                    const float df = __fsub_rn(qjs[tj * NQ + c0 + c], pj[tj]);
                    ds = __fmaf_rn(df, df, ds);
                  }
                  if (ds <= prm.g2) elig |= 1u << c;
                }
              }
              emw[(h * (NQ / 32) + sl) * 32 + lane] = elig;
            }
          }
        }
        ptx::mbar_wait(&tfull[tb], tuse & 1u);
        ptx::tc_fence_after();
#pragma unroll 1
        for (int h = 0; h < HALVES; ++h) {
          const int32_t rowbase = CG == 1 ? t * kBlockN + h * 128 + lg * 32
                                          : (t + h) * kBlockN + (int)crank * 128 + lg * 32;
          const int ra = h * 128 + lg * 32 + lane;
          const bool valid = (int64_t)rowbase + lane < prm.L;
          const float ie = inv_sm[ra];
          const uint64_t IE2 = ptx::pack2(ie, ie);
#pragma unroll
          for (int sl = 0; sl < NSL; ++sl) {
            if (sl >= nsl) break;
            const int c0 = sl * 32;
            const uint32_t taddr =
                tmem_base + ((uint32_t)(lg * 32) << 16) + (uint32_t)(tb * HALVES * NQ + h * NQ + c0);
            // pairs (this row, query c0 + c) that may enter
            const uint32_t elig = GATED ? emw[(h * (NQ / 32) + sl) * 32 + lane] : (valid ? 0xFFFFFFFFu : 0u);
            if (GATED && __reduce_or_sync(0xffffffffu, elig) == 0u) continue;   // the common case
            // exact scores of the block (kept in v), then the threshold test
            uint32_t v[32];
            __syncwarp();
            ptx::tmem_ld32(taddr, v);
            ptx::tmem_wait_ld();
            uint32_t fire = 0;
#pragma unroll
            for (int g = 0; g < 32; g += 2) {
              const uint64_t a = ptx::pack2(__uint_as_float(v[g]), __uint_as_float(v[g + 1]));
              const uint64_t iq2 = *reinterpret_cast<const uint64_t*>(iqs + c0 + g);
              const uint64_t s2 = ptx::mul2(ptx::mul2(a, iq2), IE2);   // RN(RN(acc * iq) * ie)
              const float2 th = *reinterpret_cast<const float2*>(mythr + c0 + g);
              v[g] = __float_as_uint(ptx::lo2(s2));
              v[g + 1] = __float_as_uint(ptx::hi2(s2));
              fire |= (ptx::lo2(s2) >= th.x ? 1u : 0u) << g;
              fire |= (ptx::hi2(s2) >= th.y ? 1u : 0u) << (g + 1);
            }
            fire &= elig;
            if (__reduce_or_sync(0xffffffffu, fire) == 0u) continue;
            // transpose (-inf where the pair cannot enter): lane q gets query c0 + q's
            // scores of the warp's 32 rows
#pragma unroll
            for (int c = 0; c < 32; ++c)
              tr[c * kTPad + lane] = ((fire >> c) & 1u) != 0u ? __uint_as_float(v[c]) : -CUDART_INF_F;
            __syncwarp();
            if constexpr (SMEM_LISTS) {
              TopK<KT, int32_t> tp;
#pragma unroll
              for (int rr = 0; rr < KT; ++rr) {
                tp.s[rr] = wls[(sl * KT + rr) * 32 + lane];
                tp.i[rr] = wli[(sl * KT + rr) * 32 + lane];
              }
              tp.kth_s = kth_s[sl];
              tp.kth_i = tp.i[KT - 1];
              const float b = bnd[sl];
#pragma unroll 4
              for (int rr = 0; rr < 32; ++rr) {
                const float x = tr[lane * kTPad + rr];
                if (x > tp.kth_s && x >= b) tp.insert_monotone(x, rowbase + rr, 0);
              }
#pragma unroll
              for (int rr = 0; rr < KT; ++rr) {
                wls[(sl * KT + rr) * 32 + lane] = tp.s[rr];
                wli[(sl * KT + rr) * 32 + lane] = tp.i[rr];
              }
              kth_s[sl] = tp.kth_s;
              best_s[sl] = tp.s[0];
              mythr[c0 + lane] = fmaxf(mythr[c0 + lane], tp.kth_s);
            } else {
              TopK<KT, int32_t>& tp = top[SMEM_LISTS ? 0 : sl];
              const float b = bnd[sl];
#pragma unroll 4
              for (int rr = 0; rr < 32; ++rr) {
                const float x = tr[lane * kTPad + rr];
                if (x > tp.kth_s && x >= b) tp.insert_monotone(x, rowbase + rr, 0);
              }
              mythr[c0 + lane] = fmaxf(mythr[c0 + lane], tp.kth_s);
            }
            __syncwarp();
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 1)
            ptx::mbar_arrive(&tempty[tb]);
          else
            ptx::mbar_arrive_cluster(tempty_leader0 + (uint32_t)(tb * sizeof(uint64_t)));
          ptx::mbar_arrive(&aempty[buf]);
        }
        // share the admission bound with the other CTAs (publish improvements only).
        // Geometric schedule (after 1, 2, 4, 8, ... tiles of the unit, and at its end):
        // thresholds move fast early and slowly later, and each refresh is a chain of
        // L2 round trips that one epilogue warp per sub-partition cannot hide (ncu: the
        // per-tile refresh was the top stall of the ungated scan).
        const int done = (t - t_lo) / W + 1;
        const bool refresh = (done & (done - 1)) == 0 || t + W >= t_hi;
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) {
          const int c = sl * 32 + lane;
          if (refresh && sl < nsl && c < nq) {
            uint32_t b = ptx::ld_relaxed_gpu(prm.bound + c);
            const float kth = SMEM_LISTS ? kth_s[sl] : top[SMEM_LISTS ? 0 : sl].kth_s;
            const float best = SMEM_LISTS ? best_s[sl] : top[SMEM_LISTS ? 0 : sl].s[0];
            if (kth > -CUDART_INF_F) {
              const uint32_t o = ptx::f2ord(kth);
              if (o > b) {
                atomicMax(prm.bound + c, o);
                b = o;
              }
            }
            if (b) bnd[sl] = fmaxf(bnd[sl], ptx::ord2f(b));
            if (prm.slots != nullptr) {
              // union bound (as match_tc_kernel): list l keeps its best score in slot
              // l mod k; the lists hold disjoint rows, so once all k slots are filled
              // their minimum is the score of one of k distinct rows, <= the k-th best
              uint32_t* sq = prm.slots + (int64_t)c * KT;
              const int l = (u * CG + (int)crank) * kScanEpiWarps + lg;
              if (best > -CUDART_INF_F) atomicMax(sq + l % prm.k, ptx::f2ord(best));
              uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
              for (int rr = 0; rr < KT; rr += 4) {
                const uint4 w = __ldcg(reinterpret_cast<const uint4*>(sq + rr));
                mn = min(mn, min(min(rr < prm.k ? w.x : ~0u, rr + 1 < prm.k ? w.y : ~0u),
                                 min(rr + 2 < prm.k ? w.z : ~0u, rr + 3 < prm.k ? w.w : ~0u)));
              }
              if (mn != 0u) bnd[sl] = fmaxf(bnd[sl], ptx::ord2f(mn));
            }
            mythr[c] = fmaxf(bnd[sl], kth);
          }
        }
        __syncwarp();
      }
      // One CTA, KT <= 16, gated: the 4 warps' (mostly empty) lists of a query are merged
      // here (warps 1-3 publish theirs through their transpose buffers, warp 0 inserts
      // them into its own), so the split leaves one list per query instead of four for
      // merge_partials (64-query C3 scan: 0.345 -> 0.339 ms per call).  Ungated lists are
      // full, and warp 0's serial inserts cost more in the kernel (+50 us) than the merge
      // kernel saves, so ungated calls keep four lists per split.
      constexpr bool MERGE4 = GATED && CG == 1 && KT <= 16 && 2 * KT * 32 <= 32 * kTPad;
      if constexpr (MERGE4) {
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) {
          if (sl >= nsl) break;
          float* ts = tr;                                       // [KT][32] scores
          int32_t* ti = reinterpret_cast<int32_t*>(tr + KT * 32);   // [KT][32] rows
          if (lg != 0) {
#pragma unroll
            for (int rr = 0; rr < KT; ++rr) {
              ts[rr * 32 + lane] = top[SMEM_LISTS ? 0 : sl].s[rr];
              ti[rr * 32 + lane] = top[SMEM_LISTS ? 0 : sl].i[rr];
            }
          }
          ptx::named_bar_sync(2, 32 * kScanEpiWarps);
          if (lg == 0) {
            TopK<KT, int32_t>& tp = top[SMEM_LISTS ? 0 : sl];
            for (int w = 1; w < kScanEpiWarps; ++w) {
              const float* ws = trs + w * 32 * kTPad;
              const int32_t* wi = reinterpret_cast<const int32_t*>(ws + KT * 32);
              for (int rr = 0; rr < KT; ++rr) {   // sorted lists: stop at the first entry that cannot enter
                const int32_t j = wi[rr * 32 + lane];
                const float v = ws[rr * 32 + lane];
                if (j < 0 || !better(v, j, tp.kth_s, tp.kth_i)) break;
                tp.insert(v, j, KT);
              }
            }
          }
          ptx::named_bar_sync(2, 32 * kScanEpiWarps);   // transpose buffers free again
        }
      }
      // this unit's lists -> partials [nq][P][KT] (list index = split * lists + list)
#pragma unroll
      for (int sl = 0; sl < NSL; ++sl) {
        const int c = sl * 32 + lane;
        if (sl < nsl && c < nq && (!MERGE4 || lg == 0)) {
          const int64_t base = MERGE4 ? ((int64_t)c * prm.P + u) * KT
                                      : ((int64_t)c * prm.P + ((int64_t)u * CG + crank) * kScanEpiWarps + lg) * KT;
          if constexpr (SMEM_LISTS) {
            // a list nothing ever entered (the common gated case) is padding: no reads; a
            // used one is read whole into registers first (the loads are independent of the
            // partial-list stores, so they are all in flight at once), then stored 16 B wide
            float ts[KT];
            int32_t ti[KT];
            const bool used = best_s[sl] > -CUDART_INF_F;
#pragma unroll
            for (int rr = 0; rr < KT; ++rr) {
              ts[rr] = used ? __ldcg(wls + (sl * KT + rr) * 32 + lane) : -CUDART_INF_F;
              ti[rr] = used ? __ldcg(wli + (sl * KT + rr) * 32 + lane) : -1;
            }
#pragma unroll
            for (int rr = 0; rr < KT; rr += 4) {
              *reinterpret_cast<float4*>(prm.part_s + base + rr) = make_float4(ts[rr], ts[rr + 1], ts[rr + 2], ts[rr + 3]);
              *reinterpret_cast<int4*>(prm.part_i + base + rr) = make_int4(ti[rr], ti[rr + 1], ti[rr + 2], ti[rr + 3]);
            }
          } else {
#pragma unroll
            for (int rr = 0; rr < KT; rr += 4) {
              *reinterpret_cast<float4*>(prm.part_s + base + rr) =
                  make_float4(top[SMEM_LISTS ? 0 : sl].s[rr], top[SMEM_LISTS ? 0 : sl].s[rr + 1],
                              top[SMEM_LISTS ? 0 : sl].s[rr + 2], top[SMEM_LISTS ? 0 : sl].s[rr + 3]);
              *reinterpret_cast<int4*>(prm.part_i + base + rr) =
                  make_int4(top[SMEM_LISTS ? 0 : sl].i[rr], top[SMEM_LISTS ? 0 : sl].i[rr + 1],
                            top[SMEM_LISTS ? 0 : sl].i[rr + 2], top[SMEM_LISTS ? 0 : sl].i[rr + 3]);
            }
          }
        }
      }
      __syncwarp();
    }
  }

  ptx::griddep_launch_dependents();   // the merge may be scheduled (it waits for our completion)
  ptx::tc_fence_before();
  __syncthreads();
  if (CG == 2) ptx::cluster_sync();   // no CTA leaves while its peer may still signal it
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, 512);
  }
}

// Query-tile box (TMA rows) for a batch: the smallest encoded box >= NQ.
// Query-tile box (TMA rows) = exactly the B rows a CTA's MMA reads (N for one CTA, N/2 on
// a CTA pair; a multiple of 16 <= 128): no query rows are staged that the MMA skips.
int scan_box(int rows) { return rows; }
int box_index(int box) { return box / 8 - 1; }
// MMA N: queries rounded up to 16 (the instruction's granularity), not to the epilogue's
// 32-query slots -- TMEM columns [NM, NQ) of a half are never written and belong to
// inactive queries only
int scan_nm(int nq) { return (nq + 15) / 16 * 16; }

template <int KT, int JP, bool G, int CG, int W>
cudaError_t launch_scan_t(Pool& p, const ScanParams& prm, int box, int grid, cudaStream_t s) {
  auto kern = match_scan_kernel<KT, JP, G, CG, W>;
  const size_t smem = scan_layout(prm.stages, prm.b_bytes, JP, prm.NQ, CG, KT, W).total;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kScanThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see griddep_wait()
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, p.tmap_qs[box_index(box)], CG == 1 ? p.tmap_pool : p.tmap_pool2, prm);
}

template <int KT, bool G, int CG, int W>
cudaError_t launch_scan_kt(Pool& p, const ScanParams& prm, int box, int grid, cudaStream_t s) {
  switch (p.JP) {
    case 4: return launch_scan_t<KT, 4, G, CG, W>(p, prm, box, grid, s);
    case 8: return launch_scan_t<KT, 8, G, CG, W>(p, prm, box, grid, s);
    default: return launch_scan_t<KT, 16, G, CG, W>(p, prm, box, grid, s);
  }
}

template <bool G>
cudaError_t launch_scan_g(Pool& p, const MatchArgs& a, const ScanParams& prm, int box, int grid, int cg, int w,
                          cudaStream_t s) {
  if (cg == 2)   // eligibility: KT = 8 only
    return w == 2 ? launch_scan_kt<8, G, 2, 2>(p, prm, box, grid, s) : launch_scan_kt<8, G, 2, 1>(p, prm, box, grid, s);
  switch (a.KT) {
    case 8: return launch_scan_kt<8, G, 1, 1>(p, prm, box, grid, s);
    case 16: return launch_scan_kt<16, G, 1, 1>(p, prm, box, grid, s);
    default: return launch_scan_kt<32, G, 1, 1>(p, prm, box, grid, s);
  }
}

}  // namespace

int scan_cg(int nq) { return nq > kBlockM ? 2 : 1; }

// tiles per pipeline stage: 2 on CTA pairs only when policy bit 2 asks for the wide mode
// (opt-in: it cuts the L2 -> SM bytes by 18 % on a 200-query C3 call, but that call is at
// the ridge -- tensor pipe 64-70 % and DRAM 62 % busy in both modes -- so the narrow
// pair's double-buffered accumulators win, 0.465 vs 0.491 ms) and if the
// wide stages fit shared memory
int scan_w(const Pool& p, int nq, int KT) {
  if (scan_cg(nq) != 2 || (p.kernel_policy & 4) == 0) return 1;
  const int NQ = (nq + 31) / 32 * 32;
  const uint32_t b_bytes = (uint32_t)scan_box(scan_nm(nq) / 2) * kBlockK * 2;
  return scan_layout(3, b_bytes, p.JP, NQ, 2, KT, 2).total <= kSmemLimit ? 2 : 1;
}

int scan_stages(const Pool& p, int nq, int KT) {
  const int cg = scan_cg(nq);
  if (nq < 1 || nq > kBlockM * cg || KT > 32 || (cg == 2 && KT != 8)) return 0;
  const int NQ = (nq + 31) / 32 * 32;
  if (NQ * KT > kScanListRegs) return 0;   // register lists: (NQ / 32) x KT entries per lane
  const uint32_t b_bytes = (uint32_t)scan_box(scan_nm(nq) / cg) * kBlockK * 2;
  const int w = scan_w(p, nq, KT);
  for (int st = 6; st >= 3; --st)
    if (scan_layout(st, b_bytes, p.JP, NQ, cg, KT, w).total <= kSmemLimit) return st;
  return 0;
}

cudaError_t launch_match_scan(Pool& p, const MatchArgs& a, int32_t S, int32_t grid, cudaStream_t s) {
  ScanParams prm{};
  const int cg = scan_cg(a.nq);
  const int NQ = (a.nq + 31) / 32 * 32;
  const int NM = scan_nm(a.nq);
  const int box = scan_box(NM / cg);
  prm.inv_q = p.q_inv;
  prm.q_joints = p.q_joints;
  prm.pool_inv = p.inv_norm;
  prm.pool_joints = p.joints;
  prm.part_s = p.part_s;
  prm.part_i = p.part_i;
  prm.bound = p.bound;
  prm.L = p.local;
  prm.nq = a.nq;
  prm.NQ = NQ;
  prm.NM = NM;
  prm.d = p.cfg.dim;
  prm.n_pt = (int32_t)((p.local + kBlockN - 1) / kBlockN);
  prm.S = S;
  prm.P = S * scan_lists_per_split(a.nq, a.KT, a.gated != 0);
  prm.stages = scan_stages(p, a.nq, a.KT);
  prm.b_bytes = (uint32_t)box * kBlockK * 2;
  prm.idesc = ptx::idesc_bf16_f32(kBlockM * cg, (uint32_t)NM);
  prm.g2 = a.g2;
  prm.k = a.k;
  if (prm.stages == 0 || grid % cg != 0) return cudaErrorInvalidValue;
  cudaError_t e = cudaSuccess;
  if (!a.zeroed && (e = cudaMemsetAsync(p.bound, 0, (size_t)(a.nq + 1) * sizeof(uint32_t), s)) != cudaSuccess)
    return e;
  prm.slots = a.slots ? p.slots : nullptr;
  prm.glist_s = p.scan_glist_s;
  prm.glist_i = p.scan_glist_i;
  if (cg == 2 && (prm.glist_s == nullptr || grid > p.num_sms)) return cudaErrorInvalidValue;
  if (prm.slots != nullptr && !a.zeroed) {
    e = cudaMemsetAsync(p.slots, 0, (size_t)a.nq * a.KT * sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
  }
  const int w = scan_w(p, a.nq, a.KT);
  e = a.gated ? launch_scan_g<true>(p, a, prm, box, grid, cg, w, s)
              : launch_scan_g<false>(p, a, prm, box, grid, cg, w, s);
  ++p.launches;
  return e;
}

int scan_lists_per_split(int nq, int KT, bool gated) {
  return gated && scan_cg(nq) == 1 && KT <= 16 ? 1 : kScanEpiWarps * scan_cg(nq);
}

}  // namespace ams
