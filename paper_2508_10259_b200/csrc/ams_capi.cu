// ams_capi.cu -- the C ABI (include/ams.h): pool lifecycle, record, match, shard
// exchange over NCCL, instrumentation.  Every entry point returns ams_status_t and
// never throws.
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only; ranges cost a pointer check unless a profiler is attached

#include "ams_internal.cuh"

using ams::Pool;

namespace {
// host-side NVTX range around an entry point (nsys / ncu --nvtx show the call structure)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

struct ams_pool_s {
  Pool p;
};

namespace {

#define AMS_CUDA_TRY(expr)                    \
  do {                                        \
    cudaError_t e_ = (expr);                  \
    if (e_ != cudaSuccess) {                  \
      if (getenv("AMS_LOG"))                  \
        fprintf(stderr, "[ams] %s:%d %s: %s\n", __FILE__, __LINE__, #expr, cudaGetErrorString(e_)); \
      return fail(pool, AMS_ERR_CUDA);        \
    }                                         \
  } while (0)

inline ams_status_t fail(ams_pool_s* pool, ams_status_t st) {
  if (pool != nullptr && (st == AMS_ERR_CUDA || st == AMS_ERR_NCCL) && !pool->p.broken) {
    pool->p.broken = true;
    pool->p.broken_st = st;
  }
  return st;
}

// Sticky pool status: an earlier failure, or a peer-exchange wait that timed out (the
// consumer kernel sets the host-mapped error word; no synchronisation needed to read it).
inline ams_status_t pool_status(ams_pool_s* pool) {
  ams::Pool& p = pool->p;
  if (!p.broken && p.x_err_host != nullptr && *static_cast<volatile unsigned int*>(p.x_err_host) != 0)
    fail(pool, AMS_ERR_NCCL);
  return p.broken ? p.broken_st : AMS_OK;
}

// Is `s` being captured into a CUDA graph?  (Capture forbids the pageable host copies and
// the host epoch counter of the peer exchange.)
inline bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

// Host-append staging is allocated on the first host-sourced append, with a fixed byte
// budget (not sized by the pool: device-sourced appends never need it).
constexpr size_t kStageBytes = (size_t)64 << 20;

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                       CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                       CUtensorMapFloatOOBfill);

PFN_encodeTiled_t get_encode() {
  static PFN_encodeTiled_t fn = nullptr;
  if (fn == nullptr) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(f);
  }
  return fn;
}

// 2-D bf16 K-major tile map: rows x d, box {64, box_rows}, 128-B swizzle, OOB -> 0
bool encode_bf16_map(CUtensorMap* m, void* base, int64_t rows, int32_t d, uint32_t box_rows) {
  PFN_encodeTiled_t enc = get_encode();
  if (enc == nullptr) return false;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {(cuuint32_t)ams::kBlockK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// small-batch kernel: query tiles of exactly 8, 16, ..., 128 rows (box i = 8 (i + 1)): the
// MMA's N (queries rounded up to 16) on one CTA, or its half on a CTA pair
bool encode_query_boxes(ams::Pool& p, int32_t d) {
  for (int i = 0; i < 16; ++i)
    if (!encode_bf16_map(&p.tmap_qs[i], p.q_stage, p.q_pad, d, (uint32_t)(8 * (i + 1)))) return false;
  return true;
}

bool is_device_ptr(const void* ptr) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// Smallest gated bf16 batch staged in (joint 0, joint 1) order (below it one warp's queries span
// most of the joint range and the per-lane packed filter is cheaper).
constexpr int32_t kSortMinQueries = 129;

size_t esize(const Pool& p) { return p.cfg.dtype == AMS_DTYPE_BF16 ? 2 : 4; }

// Plan of the tcgen05 kernel.  Queries > 128 -> CTA pairs (cta_group::2, 256-query
// tiles, 2x the operand reuse per byte from L2); otherwise one CTA per 128-query tile
// (the HBM-bound scan).  Row splits S: units = n_qt * S are dealt round-robin to the
// persistent clusters; minimise the busiest cluster's tile count
// ceil(U / clusters) * ceil(n_pt / S), ties -> fewer splits (fewer partial lists).
void plan_tc(const Pool& p, int nq, int KT, int& S, int& grid, int& cg, int& cl) {
  cg = nq > ams::kBlockM ? 2 : 1;
  const int qtile = ams::tc_query_tile(cg);
  const int n_qt = (nq + qtile - 1) / qtile;
  const int64_t n_pt = (p.local + ams::kBlockN - 1) / ams::kBlockN;
  // Opt-in (policy bit 1): two CTA pairs per 4-CTA cluster share (multicast) the pool
  // rows when the query tiles pair up.  Off by default: clusters must fit within a GPC
  // and only 33 four-CTA clusters (132 of 148 SMs) are co-resident on a B200; the grid is
  // limited to them because the wave lockstep needs the whole grid resident.  Measured
  // at the 1 kW cap: +9.5 % per SM (clock 1305 -> 1425 MHz) but -10.8 % SMs, net -2.4 %.
  cl = (cg == 2 && n_qt % 2 == 0 && p.max_clusters4 >= 1 && (p.kernel_policy & 2) != 0) ? 4 : cg;
  const int clusters = std::min(p.num_sms / cl, std::max(1, cl == 4 ? p.max_clusters4 : cl == 2 ? p.max_clusters2
                                                                                               : p.num_sms));
  const int n_qg = n_qt / (cl / cg);   // units per row split
  const int64_t nq_pad = (int64_t)n_qt * qtile;
  int64_t s_cap = std::max<int64_t>(1, p.part_cap / (nq_pad * ams::kEpiHalves * KT));
  s_cap = std::min<int64_t>(s_cap, std::max<int64_t>(1, n_pt));
  s_cap = std::min<int64_t>(s_cap, std::max<int64_t>(1, (int64_t)64 * clusters / n_qg + 1));
  int64_t best_cost = LLONG_MAX;
  int best = 1;
  for (int64_t s = 1; s <= s_cap; ++s) {
    const int64_t U = (int64_t)n_qg * s;
    const int64_t waves = (U + clusters - 1) / clusters;
    const int64_t per = (n_pt + s - 1) / s;
    const int64_t cost = waves * per * 64 + s;  // + small penalty per split (merge work)
    if (cost < best_cost) {
      best_cost = cost;
      best = (int)s;
    }
  }
  S = best;
  grid = (int)std::min<int64_t>((int64_t)n_qg * S, clusters) * cl;
}

// Plan of the small-batch kernel: one query tile, so units are row splits only; same
// cost model as plan_tc (busiest CTA's tile count, ties -> fewer splits).
void plan_scan(const Pool& p, int nq, int KT, bool gated, int& S, int& grid) {
  const int w = ams::scan_w(p, nq, KT);   // splits are counted in super-tiles of w tiles
  const int64_t n_pt = ((p.local + ams::kBlockN - 1) / ams::kBlockN + w - 1) / w;
  const int cg = ams::scan_cg(nq);
  const int ctas = std::min(p.num_sms / cg, cg == 2 ? std::max(1, p.max_clusters2) : p.num_sms);   // tiles in flight
  const int64_t per_split = (int64_t)nq * ams::scan_lists_per_split(nq, KT, gated) * KT;
  int64_t s_cap = std::max<int64_t>(1, p.part_cap / per_split);
  s_cap = std::min<int64_t>({s_cap, std::max<int64_t>(1, n_pt), (int64_t)8 * ctas});
  int64_t best_cost = LLONG_MAX;
  int best = 1;
  for (int64_t s = 1; s <= s_cap; ++s) {
    const int64_t cost = ((s + ctas - 1) / ctas) * ((n_pt + s - 1) / s) * 64 + s;
    if (cost < best_cost) {
      best_cost = cost;
      best = (int)s;
    }
  }
  S = best;
  grid = (int)std::min<int64_t>(S, ctas) * cg;
}

void plan_simt(const Pool& p, int nq, int KT, int& S) {
  const int64_t per_split = (int64_t)nq * ams::kSimtThreads * KT;
  int64_t s_cap = std::max<int64_t>(1, p.part_cap / per_split);
  int64_t want = std::max<int64_t>(1, (2 * p.num_sms + nq - 1) / nq);
  want = std::min<int64_t>(want, std::max<int64_t>(1, p.local / ams::kSimtThreads));
  S = (int)std::max<int64_t>(1, std::min(want, s_cap));
}

void free_peers(Pool& p) {
  if (p.peer_mode)
    for (int g = 0; g < p.peers.G; ++g)
      if (g != p.peers.rank) {
        if (p.peers.s[g]) cudaIpcCloseMemHandle(p.peers.s[g]);
        if (p.peers.i[g]) cudaIpcCloseMemHandle(p.peers.i[g]);
        if (p.peers.flag[g]) cudaIpcCloseMemHandle(p.peers.flag[g]);
      }
  void* own[] = {p.x_s, p.x_i, p.x_flag, p.x_done, p.x_barrier};
  for (void* q : own)
    if (q) cudaFree(q);
  // the error word outlives the peer mode only if it fired (pool_status keeps reporting it)
  if (p.x_err_host && *static_cast<volatile unsigned int*>(p.x_err_host) == 0) {
    cudaFreeHost(p.x_err_host);
    p.x_err_host = nullptr;
  }
  p.peer_mode = false;
  p.peers = ams::PeerTable{};
  p.x_s = nullptr;
  p.x_i = nullptr;
  p.x_flag = nullptr;
  p.x_done = nullptr;
  p.x_barrier = nullptr;
}

void free_all(Pool& p) {
  free_peers(p);
  if (p.x_err_host) cudaFreeHost(p.x_err_host);
  p.x_err_host = nullptr;
  for (int b = 0; b < 2; ++b) {
    if (p.staged[b]) cudaEventDestroy(p.staged[b]);
    if (p.consumed[b]) cudaEventDestroy(p.consumed[b]);
    p.staged[b] = p.consumed[b] = nullptr;
  }
  if (p.copy_stream) cudaStreamDestroy(p.copy_stream);
  p.copy_stream = nullptr;
  if (p.est_ready) cudaEventDestroy(p.est_ready);
  if (p.est_host) cudaFreeHost(p.est_host);
  p.est_ready = nullptr;
  p.est_host = nullptr;
  void* ptrs[] = {p.scan_glist_s, p.scan_glist_i, p.emb, p.inv_norm, p.joints, p.q_stage, p.q_inv, p.q_joints,
                  p.q_joints_raw[0], p.q_joints_raw[1],
                  p.q_raw[0], p.q_raw[1], p.q_perm, p.bound, p.slots,
                  p.gf_cnt, p.gf_cand, p.gf_qbins, p.snap_j, p.snap_id, p.snap_off, p.snap_aux,
                  p.part_s, p.part_i, p.shard_s, p.shard_i, p.gath_s, p.gath_i, p.stage_emb,
                  p.stage_joints, p.est_dev};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  for (auto& e : p.ev_free) cudaEventDestroy(e);
  for (auto& e : p.ev_pending) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  p.ev_free.clear();
  p.ev_pending.clear();
}

}  // namespace

extern "C" {

int32_t ams_abi_version(void) { return AMS_ABI_VERSION; }

#ifndef AMS_BUILD_ID
#define AMS_BUILD_ID "unknown"
#endif
const char* ams_build_id(void) { return AMS_BUILD_ID; }

const char* ams_status_string(ams_status_t st) {
  switch (st) {
    case AMS_OK: return "AMS_OK";
    case AMS_ERR_INVALID_ARGUMENT: return "AMS_ERR_INVALID_ARGUMENT";
    case AMS_ERR_CAPACITY: return "AMS_ERR_CAPACITY";
    case AMS_ERR_OUT_OF_MEMORY: return "AMS_ERR_OUT_OF_MEMORY";
    case AMS_ERR_CUDA: return "AMS_ERR_CUDA";
    case AMS_ERR_NCCL: return "AMS_ERR_NCCL";
    case AMS_ERR_UNSUPPORTED: return "AMS_ERR_UNSUPPORTED";
    case AMS_ERR_INTERNAL: return "AMS_ERR_INTERNAL";
  }
  return "AMS_ERR_UNKNOWN";
}

ams_status_t ams_shard_locate(int64_t capacity, int32_t world, int64_t shard_block, int64_t global_index,
                              int32_t* owner, int64_t* local_row) {
  if (capacity < 0 || world < 1 || shard_block < 0 || global_index < 0 || global_index >= capacity)
    return AMS_ERR_INVALID_ARGUMENT;
  const int64_t B = ams::shard_block_size(capacity, world, shard_block);
  if (owner) *owner = ams::shard_owner(global_index, world, B);
  if (local_row) *local_row = ams::shard_local(global_index, world, B);
  return AMS_OK;
}

ams_status_t ams_shard_capacity(int64_t capacity, int32_t world, int64_t shard_block, int32_t rank,
                                int64_t* rows) {
  if (capacity < 0 || world < 1 || shard_block < 0 || rank < 0 || rank >= world || rows == nullptr)
    return AMS_ERR_INVALID_ARGUMENT;
  const int64_t B = ams::shard_block_size(capacity, world, shard_block);
  *rows = ams::shard_count(capacity, rank, world, B);
  return AMS_OK;
}

ams_status_t ams_get_nccl_unique_id(void* out128) {
  if (out128 == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return AMS_ERR_NCCL;
  memcpy(out128, &id, sizeof id);
  return AMS_OK;
}

ams_status_t ams_pool_create(const ams_pool_config_t* cfg, ams_pool_t* out) {
  ams_pool_s* pool = nullptr;
  if (cfg == nullptr || out == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  const auto& c = *cfg;
  if (c.dim < 64 || c.dim > 16384 || c.dim % 64 != 0) return AMS_ERR_INVALID_ARGUMENT;
  if (c.joint_dim < 1 || c.joint_dim > 16) return AMS_ERR_INVALID_ARGUMENT;
  if (c.dtype != AMS_DTYPE_BF16 && c.dtype != AMS_DTYPE_FP32) return AMS_ERR_INVALID_ARGUMENT;
  if (c.capacity < 0 || c.max_queries < 1 || c.max_k < 1 || c.max_k > 64) return AMS_ERR_INVALID_ARGUMENT;
  if (c.world < 1 || c.world > 64 || c.rank < 0 || c.rank >= c.world || c.shard_block < 0)
    return AMS_ERR_INVALID_ARGUMENT;
  if (c.world > 1 && c.nccl_id == nullptr) return AMS_ERR_INVALID_ARGUMENT;

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || c.device < 0 || c.device >= ndev) {
    cudaGetLastError();
    return AMS_ERR_INVALID_ARGUMENT;
  }
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, c.device) != cudaSuccess) return AMS_ERR_CUDA;
  if (prop.major != 10 || prop.minor != 0) return AMS_ERR_UNSUPPORTED;  // built for sm_100a only
  if (cudaSetDevice(c.device) != cudaSuccess) return AMS_ERR_CUDA;

  pool = new (std::nothrow) ams_pool_s;
  if (pool == nullptr) return AMS_ERR_OUT_OF_MEMORY;
  Pool& p = pool->p;
  p.cfg = c;
  p.cfg.nccl_id = nullptr;
  p.num_sms = prop.multiProcessorCount;
  p.max_clusters2 = ams::tc_max_active_clusters(2);
  p.max_clusters4 = ams::tc_max_active_clusters(4);
  p.JP = c.joint_dim <= 4 ? 4 : c.joint_dim <= 8 ? 8 : 16;
  p.B = ams::shard_block_size(c.capacity, c.world, c.shard_block);
  p.cap_shard = ams::shard_count(c.capacity, c.rank, c.world, p.B);
  if (p.cap_shard >= ((int64_t)1 << 31) - ams::kRowAlign) {
    delete pool;
    return AMS_ERR_INVALID_ARGUMENT;  // local row ids are int32 inside the kernels
  }
  p.cap_pad = round_up(std::max<int64_t>(p.cap_shard, 1), ams::kRowAlign);
  p.KT_max = ams::pick_KT(c.max_k);
  p.q_pad = (int32_t)round_up(c.max_queries, 2 * ams::kBlockM);
  const size_t es = esize(p);
  const int32_t d = c.dim;

  auto alloc = [&](void** ptr, size_t bytes) -> bool {
    if (cudaMalloc(ptr, std::max<size_t>(bytes, 16)) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return cudaMemset(*ptr, 0, std::max<size_t>(bytes, 16)) == cudaSuccess;
  };
  // partial-list workspace: tcgen05 path needs q_pad * 2 * S * KT, S bounded by the
  // pool's tile count and by ~64 waves of units; SIMT path q * 128 * S * KT.
  const int64_t n_pt_max = p.cap_pad / ams::kBlockN;
  int64_t part = 0;
  if (c.dtype == AMS_DTYPE_BF16) {
    const int64_t s_max = std::min<int64_t>(n_pt_max, (int64_t)64 * p.num_sms + 1);
    part = std::min<int64_t>((int64_t)p.q_pad * s_max, (int64_t)ams::kBlockM * 64 * p.num_sms + p.q_pad) *
           ams::kEpiHalves * p.KT_max;
    // the small-batch kernel keeps 4 (8 on a CTA pair) lists per row split for nq <= 256
    part = std::max<int64_t>(part, (int64_t)std::min(p.q_pad, 256) * 8 * p.KT_max * std::min<int64_t>(n_pt_max, 8));
  } else {
    const int64_t s_max = std::max<int64_t>(1, std::min<int64_t>(p.cap_pad / ams::kSimtThreads, 2 * p.num_sms));
    part = std::min<int64_t>((int64_t)c.max_queries * s_max, (int64_t)c.max_queries + 2 * p.num_sms) *
           ams::kSimtThreads * p.KT_max;
  }
  p.part_cap = part;
  p.stage_rows = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(c.capacity, 1),
                                                        (int64_t)(kStageBytes / ((size_t)d * es + 4 * c.joint_dim))));
  bool ok = alloc(&p.emb, (size_t)p.cap_pad * d * es) && alloc((void**)&p.inv_norm, (size_t)p.cap_pad * 4) &&
            alloc((void**)&p.joints, (size_t)p.cap_pad * p.JP * 4) &&
            alloc(&p.q_stage, (size_t)p.q_pad * d * es) && alloc((void**)&p.q_inv, (size_t)p.q_pad * 4) &&
            alloc((void**)&p.q_joints, (size_t)p.q_pad * p.JP * 4) &&
            alloc((void**)&p.q_joints_raw[0], (size_t)c.max_queries * c.joint_dim * 4) &&
            alloc((void**)&p.q_joints_raw[1], (size_t)c.max_queries * c.joint_dim * 4) &&
            alloc(&p.q_raw[0], (size_t)c.max_queries * d * es) && alloc(&p.q_raw[1], (size_t)c.max_queries * d * es) &&
            alloc((void**)&p.q_perm, (size_t)p.q_pad * 4) &&
            alloc((void**)&p.bound, (size_t)(p.q_pad + 32) * 4) &&
            alloc((void**)&p.slots, (size_t)p.q_pad * p.KT_max * 4) &&
            alloc((void**)&p.part_s, (size_t)part * 4) && alloc((void**)&p.part_i, (size_t)part * 4) &&
            alloc((void**)&p.shard_s, (size_t)c.max_queries * c.max_k * 4) &&
            alloc((void**)&p.shard_i, (size_t)c.max_queries * c.max_k * 8);
  if (ok && c.dtype == AMS_DTYPE_BF16) {
    const size_t gl = (size_t)p.num_sms * 4 * 8 * 8 * 32;   // see Pool::scan_glist_s
    ok = alloc((void**)&p.scan_glist_s, gl * 4) && alloc((void**)&p.scan_glist_i, gl * 4);
  }
  if (ok && c.dtype == AMS_DTYPE_BF16) {
    p.gf_cap = std::max(256, 8 * c.max_k);
    ok = alloc((void**)&p.gf_cnt, (size_t)p.q_pad * 4) && alloc((void**)&p.gf_cand, (size_t)p.q_pad * p.gf_cap * 4) &&
         alloc((void**)&p.gf_qbins, (size_t)(ams::kQBins + 3) * 4);
  }
  if (ok) ok = alloc((void**)&p.est_dev, 16);
  p.collective = c.world > 1 || c.nccl_id != nullptr;
  if (ok && p.collective)
    ok = alloc((void**)&p.gath_s, (size_t)c.world * c.max_queries * c.max_k * 4) &&
         alloc((void**)&p.gath_i, (size_t)c.world * c.max_queries * c.max_k * 8);
  if (!ok) {
    free_all(p);
    delete pool;
    return AMS_ERR_OUT_OF_MEMORY;
  }
  if (c.dtype == AMS_DTYPE_BF16) {
    if (!encode_bf16_map(&p.tmap_pool, p.emb, p.cap_pad, d, ams::kBlockN) ||
        !encode_bf16_map(&p.tmap_pool2, p.emb, p.cap_pad, d, ams::kBlockN / 2) ||
        !encode_bf16_map(&p.tmap_pool4, p.emb, p.cap_pad, d, ams::kBlockN / 4) ||
        !encode_bf16_map(&p.tmap_q, p.q_stage, p.q_pad, d, ams::kBlockM) ||
        !encode_query_boxes(p, d)) {
      free_all(p);
      delete pool;
      return AMS_ERR_CUDA;
    }
  }
  bool sok = cudaStreamCreateWithFlags(&p.copy_stream, cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&p.est_ready, cudaEventDisableTiming) == cudaSuccess &&
             cudaMallocHost((void**)&p.est_host, 16) == cudaSuccess;
  for (int b = 0; b < 2 && sok; ++b)
    sok = cudaEventCreateWithFlags(&p.staged[b], cudaEventDisableTiming) == cudaSuccess &&
          cudaEventCreateWithFlags(&p.consumed[b], cudaEventDisableTiming) == cudaSuccess;
  if (!sok || cudaDeviceSynchronize() != cudaSuccess) {
    cudaGetLastError();
    free_all(p);
    delete pool;
    return AMS_ERR_CUDA;
  }
  if (p.collective) {
    ncclUniqueId id;
    memcpy(&id, c.nccl_id, sizeof id);
    ncclComm_t comm;
    if (ncclCommInitRank(&comm, c.world, id, c.rank) != ncclSuccess) {
      free_all(p);
      delete pool;
      return AMS_ERR_NCCL;
    }
    p.nccl_comm = comm;
  }
  *out = pool;
  return AMS_OK;
}

ams_status_t ams_pool_append(ams_pool_t pool, const void* emb, const float* joints, int64_t n,
                             int64_t* first_index, void* stream) {
  NvtxRange nvtx("ams_pool_append");
  if (pool == nullptr || n < 0) return AMS_ERR_INVALID_ARGUMENT;
  Pool& p = pool->p;
  if (pool_status(pool) != AMS_OK) return p.broken_st;
  if (n > 0 && (emb == nullptr || joints == nullptr)) return AMS_ERR_INVALID_ARGUMENT;
  if (n > p.cfg.capacity - p.size) return AMS_ERR_CAPACITY;
  if (n == 0) {
    if (first_index) *first_index = p.size;
    return AMS_OK;
  }
  AMS_CUDA_TRY(cudaSetDevice(p.cfg.device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t es = esize(p);
  const size_t row_bytes = (size_t)p.cfg.dim * es;
  const bool dev_e = is_device_ptr(emb), dev_j = is_device_ptr(joints);
  if ((!dev_e || !dev_j) && capturing(s)) return AMS_ERR_UNSUPPORTED;   // pageable copies cannot be captured
  if ((!dev_e && p.stage_emb == nullptr) || (!dev_j && p.stage_joints == nullptr)) {
    // first host-sourced append: allocate the staging buffers (stream-ordered frees are
    // not needed: they live as long as the pool)
    AMS_CUDA_TRY(cudaStreamSynchronize(s));
    if (p.stage_emb == nullptr && cudaMalloc(&p.stage_emb, (size_t)p.stage_rows * row_bytes) != cudaSuccess) {
      cudaGetLastError();
      p.stage_emb = nullptr;
      return AMS_ERR_OUT_OF_MEMORY;
    }
    if (p.stage_joints == nullptr &&
        cudaMalloc((void**)&p.stage_joints, (size_t)p.stage_rows * p.cfg.joint_dim * 4) != cudaSuccess) {
      cudaGetLastError();
      p.stage_joints = nullptr;
      return AMS_ERR_OUT_OF_MEMORY;
    }
  }
  if (first_index) *first_index = p.size;
  for (int64_t off = 0; off < n;) {
    const int64_t m = (dev_e && dev_j) ? n - off : std::min<int64_t>(n - off, p.stage_rows);
    const void* e_src = static_cast<const uint8_t*>(emb) + off * row_bytes;
    const float* j_src = joints + off * p.cfg.joint_dim;
    if (!dev_e) {
      AMS_CUDA_TRY(cudaMemcpyAsync(p.stage_emb, e_src, m * row_bytes, cudaMemcpyDefault, s));
      e_src = p.stage_emb;
    }
    if (!dev_j) {
      AMS_CUDA_TRY(cudaMemcpyAsync(p.stage_joints, j_src, m * p.cfg.joint_dim * 4, cudaMemcpyDefault, s));
      j_src = p.stage_joints;
    }
    AMS_CUDA_TRY(ams::launch_append(p, e_src, j_src, m, p.size + off, s));
    off += m;
  }
  p.size += n;
  p.local = ams::shard_count(p.size, p.cfg.rank, p.cfg.world, p.B);
  return AMS_OK;
}

// ams_match_auto's route choice (host; SURVEY.md 8(f) f3 "select by measured pass-rate").
// The expected number of eligible rows per query comes from the exact canonical gate over
// a strided sample (<= 64 queries x <= 32768 rows, one tiny kernel): synchronously when
// there is no estimate for this gate radius yet or the shard changed size by 2x, else
// refreshed asynchronously every 64 calls (pinned D2H + event; adopted once complete).
// Cost model (ms), constants from the round-1 measurements:
//   dense      0.02 + max(2 nq L d / 1.40e15, L (2d + 4J + 4) / 6.5e12)  (sustained tensor / HBM)
//   gate-first 0.03 + nq L / 2e13 (filter ALU) + ceil(nq/256) L 4 JP / 4e12 (joint reads per
//              256-query block) + nq E 2 d / 2e12 (gathered rows of the E eligible per query)
// gate-first is taken when it is cheaper and E <= bucket capacity / 2 (no overflow rescans).
static ams_status_t auto_route(ams_pool_s* pool, const float* qj_src, int32_t nq, float g2, cudaStream_t s,
                               bool* gate_first) {
  Pool& p = pool->p;
  *gate_first = false;
  if (p.cfg.dtype != AMS_DTYPE_BF16 || std::isinf(g2) || p.local <= 0) {
    p.last_route = 0;
    return AMS_OK;
  }
  auto adopt = [&]() {
    const double pairs = (double)p.est_rows * (double)p.est_queries;
    const double rate = pairs > 0 ? (double)*p.est_host / pairs : 0.0;
    p.est_elig = rate * (double)p.local;
    p.est_valid = true;
  };
  if (p.est_pending) {
    const cudaError_t q = cudaEventQuery(p.est_ready);
    if (q == cudaSuccess) {
      p.est_pending = false;
      adopt();
    } else if (q != cudaErrorNotReady) {
      return fail(pool, AMS_ERR_CUDA);
    } else {
      cudaGetLastError();   // not-ready is not an error
    }
  }
  const bool stale = !p.est_valid || p.est_g2 != g2 || p.local > 2 * p.est_L || 2 * p.local < p.est_L;
  if (stale || (++p.est_calls % 64 == 0 && !p.est_pending)) {
    int32_t rows = 0, qs = 0;
    AMS_CUDA_TRY(ams::launch_gate_estimate(p, qj_src, nq, g2, p.est_dev, &rows, &qs, s));
    AMS_CUDA_TRY(cudaMemcpyAsync(p.est_host, p.est_dev, 8, cudaMemcpyDeviceToHost, s));
    p.est_rows = rows;
    p.est_queries = qs;
    p.est_g2 = g2;
    p.est_L = p.local;
    if (stale) {
      AMS_CUDA_TRY(cudaStreamSynchronize(s));
      p.est_pending = false;
      adopt();
    } else {
      AMS_CUDA_TRY(cudaEventRecord(p.est_ready, s));
      p.est_pending = true;
    }
  }
  const double L = (double)p.local, d = p.cfg.dim, J = p.cfg.joint_dim, n = nq, E = p.est_elig;
  const double dense = 0.02 + 1e3 * std::max(2.0 * n * L * d / 1.40e15, L * (2 * d + 4 * J + 4) / 6.5e12);
  const double gf = 0.03 + 1e3 * (n * L / 2e13 + std::ceil(n / 256.0) * L * 4 * p.JP / 4e12 + n * E * 2 * d / 2e12);
  p.last_est_ms[0] = dense;
  p.last_est_ms[1] = gf;
  *gate_first = E <= 0.5 * p.gf_cap && gf < dense;
  p.last_route = *gate_first ? 1 : 0;
  return AMS_OK;
}

static ams_status_t match_impl(ams_pool_t pool, const void* q_emb, const float* q_joints, int32_t nq, int32_t k,
                               float threshold, float gate_radius, int64_t* out_index, float* out_score,
                               uint8_t* out_hit, void* stream, bool gate_first, bool auto_select = false) {
  NvtxRange nvtx(auto_select ? "ams_match_auto" : gate_first ? "ams_match_gate_first" : "ams_match");
  if (pool == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  Pool& p = pool->p;
  if (pool_status(pool) != AMS_OK) return p.broken_st;
  if (q_emb == nullptr || q_joints == nullptr || out_index == nullptr || out_score == nullptr ||
      out_hit == nullptr)
    return AMS_ERR_INVALID_ARGUMENT;
  if (nq < 1 || nq > p.cfg.max_queries || k < 1 || k > p.cfg.max_k) return AMS_ERR_INVALID_ARGUMENT;
  if (std::isnan(threshold) || std::isnan(gate_radius) || gate_radius < 0.0f) return AMS_ERR_INVALID_ARGUMENT;
  AMS_CUDA_TRY(cudaSetDevice(p.cfg.device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);

  ams::MatchArgs a{};
  a.nq = nq;
  a.k = k;
  a.KT = ams::pick_KT(k);
  {
    volatile float g = gate_radius;
    a.g2 = g * g;  // fp32(gamma^2), reading R3
  }
  a.gated = std::isinf(a.g2) ? 0 : 1;
  a.threshold = threshold;

  // stage queries: device sources are read in place; host sources are copied on the
  // pool's copy stream into staging buffer b (free once the prep of two calls ago has
  // read it), and s waits only for that copy -- the H2D of this call overlaps whatever
  // s is still running from the previous one.
  const size_t es = esize(p);
  const void* q_src = q_emb;
  const float* qj_src = q_joints;
  const bool host_q = !is_device_ptr(q_emb), host_j = !is_device_ptr(q_joints);
  if ((host_q || host_j || (p.collective && p.peer_mode) || auto_select) && capturing(s))
    return AMS_ERR_UNSUPPORTED;   // pageable copies / the host epoch counter / the estimate sync cannot be captured
  int b = -1;
  if (host_q || host_j) {
    b = p.stage_buf;
    p.stage_buf ^= 1;
    AMS_CUDA_TRY(cudaStreamWaitEvent(p.copy_stream, p.consumed[b], 0));
    if (host_q) {
      AMS_CUDA_TRY(cudaMemcpyAsync(p.q_raw[b], q_emb, (size_t)nq * p.cfg.dim * es, cudaMemcpyDefault, p.copy_stream));
      q_src = p.q_raw[b];
    }
    if (host_j) {
      AMS_CUDA_TRY(cudaMemcpyAsync(p.q_joints_raw[b], q_joints, (size_t)nq * p.cfg.joint_dim * 4, cudaMemcpyDefault,
                                   p.copy_stream));
      qj_src = p.q_joints_raw[b];
    }
    AMS_CUDA_TRY(cudaEventRecord(p.staged[b], p.copy_stream));
    AMS_CUDA_TRY(cudaStreamWaitEvent(s, p.staged[b], 0));
  }
  if (auto_select) {
    const ams_status_t rs = auto_route(pool, qj_src, nq, a.g2, s, &gate_first);
    if (rs != AMS_OK) return rs;
  }
  // Gated batches are staged in (joint 0, joint 1) order (the epilogue's warp-level gate
  // test then rejects most columns for all 32 queries of a warp at once).  The order is
  // invisible to the caller: partial lists land at the caller's query index.
  // The small-batch kernel (pool rows on the MMA M side) needs no query order.
  // Ungated batches of 129-256 queries stay on the 256-query-tile kernel: the CTA-pair
  // small-batch kernel keeps its lists in global memory, and without a gate every list
  // fills and is re-read on inserts (C3 pool, k = 8: 0.63-0.88 ms vs 0.455 ms; gated it
  // is the faster one, 0.36-0.46 ms).  Policy bit 3 keeps them on the CTA pairs (A/B).
  const bool use_scan = !gate_first && p.cfg.dtype == AMS_DTYPE_BF16 && p.local > 0 && (p.kernel_policy & 1) == 0 &&
                        (nq <= ams::kBlockM || a.gated || (p.kernel_policy & 8) != 0) &&
                        ams::scan_stages(p, nq, a.KT) > 0 &&
                        (int64_t)nq * ams::scan_lists_per_split(nq, a.KT, a.gated != 0) * a.KT <= p.part_cap;   // >= 1 split fits
  // Gated gate-first batches of 17..1024 queries are staged in joint-0 bins instead (the
  // row kernels look up, per pool row, the queries within gamma of its joint 0).
  // (Up to 1024 queries, whose joints fit in shared memory: at 1024 the two designs are
  // even on C3's pool, and at 2048 the block kernel over the 2-D query order wins, 0.27 vs
  // 0.50 ms, so larger batches keep it.)
  const bool qbins = gate_first && p.cfg.dtype == AMS_DTYPE_BF16 && a.gated && p.local > 0 && nq > ams::kGfRowsMaxQ &&
                     nq <= ams::kGfBinnedMaxQ;
  const bool sorted =
      qbins || (p.cfg.dtype == AMS_DTYPE_BF16 && a.gated && p.local > 0 && nq >= kSortMinQueries && !use_scan);
  a.qbins = qbins ? 1 : 0;
  if (qbins)
    AMS_CUDA_TRY(ams::launch_query_order_j0(p, qj_src, nq, s));
  else if (sorted)
    AMS_CUDA_TRY(ams::launch_query_order(p, qj_src, nq, s));
  // the dense bf16 kernels start from zeroed per-query bounds (+ the K2 wave counter) and,
  // ungated, zeroed union slots: the prep kernel clears them (no memset node between it
  // and the dense kernel, which is then its programmatic dependent).  Slots: K2 indexes
  // them by padded query tile (<= round_up(nq, 256) rows), the small-batch kernel by query.
  // (gate-first: the candidate counts)
  const bool dense_bf16 = !gate_first && p.cfg.dtype == AMS_DTYPE_BF16 && p.local > 0;
  const bool gf_bf16 = gate_first && p.cfg.dtype == AMS_DTYPE_BF16;
  const int32_t zero_bound = dense_bf16 ? nq + 1 : gf_bf16 ? nq : 0;
  const int32_t zero_slots = dense_bf16 && !a.gated ? (int32_t)round_up(nq, 2 * ams::kBlockM) * a.KT : 0;
  AMS_CUDA_TRY(ams::launch_query_prep(p, q_src, qj_src, nq, sorted ? p.q_perm : nullptr, gf_bf16 ? p.gf_cnt : p.bound,
                                      zero_bound, p.slots, zero_slots, s));
  a.zeroed = dense_bf16 || gf_bf16 ? 1 : 0;
  if (b >= 0) AMS_CUDA_TRY(cudaEventRecord(p.consumed[b], s));   // staging b read (order + prep)

  const bool multi = p.collective;
  float* shard_s = multi ? p.shard_s : out_score;
  int64_t* shard_i = multi ? p.shard_i : out_index;
  uint8_t* shard_hit = multi ? nullptr : out_hit;

  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p.profiling) {
    for (int t = 0; t < 2; ++t) {
      cudaEvent_t ev;
      if (!p.ev_free.empty()) {
        ev = p.ev_free.back();
        p.ev_free.pop_back();
      } else {
        AMS_CUDA_TRY(cudaEventCreate(&ev));
      }
      (t == 0 ? e0 : e1) = ev;
    }
  }

  int32_t P = 0;
  if (gate_first && p.cfg.dtype == AMS_DTYPE_BF16) {
    if (e0) AMS_CUDA_TRY(cudaEventRecord(e0, s));
    AMS_CUDA_TRY(ams::launch_gate_first(p, a, shard_s, shard_i, shard_hit, sorted, s));
    if (e1) {
      AMS_CUDA_TRY(cudaEventRecord(e1, s));
      p.ev_pending.emplace_back(e0, e1);
    }
    p.last_kernel = 3;
    p.last_splits = 0;
    p.last_partials = 0;
    p.last_grid = 0;
  } else if (p.local > 0) {
    if (p.cfg.dtype == AMS_DTYPE_FP32 && !a.gated &&
        (int64_t)nq * ams::f32_tile_lists(p.local) * a.KT <= p.part_cap) {
      // ungated fp32: every pair is scored -- the tiled exact kernel (plan id 6)
      P = ams::f32_tile_lists(p.local);
      if (e0) AMS_CUDA_TRY(cudaEventRecord(e0, s));
      AMS_CUDA_TRY(ams::launch_match_f32_tile(p, a, s));
      if (e1) AMS_CUDA_TRY(cudaEventRecord(e1, s));
      p.last_splits = P;
      p.last_grid = P * ((nq + 15) / 16);
      p.last_kernel = 6;
    } else if (p.cfg.dtype == AMS_DTYPE_FP32) {
      int S;
      plan_simt(p, nq, a.KT, S);
      P = S * ams::kSimtThreads;
      if (e0) AMS_CUDA_TRY(cudaEventRecord(e0, s));
      AMS_CUDA_TRY(ams::launch_match_simt(p, a, S, s));
      if (e1) AMS_CUDA_TRY(cudaEventRecord(e1, s));
      p.last_splits = S;
      p.last_grid = nq * S;
      p.last_kernel = 0;
    } else if (use_scan) {
      int S, grid;
      plan_scan(p, nq, a.KT, a.gated != 0, S, grid);
      P = S * ams::scan_lists_per_split(nq, a.KT, a.gated != 0);
      a.slots = (!a.gated && P >= a.k) ? 1 : 0;   // union-bound slots (launch_match_scan)
      if (e0) AMS_CUDA_TRY(cudaEventRecord(e0, s));
      AMS_CUDA_TRY(ams::launch_match_scan(p, a, S, grid, s));
      if (e1) AMS_CUDA_TRY(cudaEventRecord(e1, s));
      p.last_splits = S;
      p.last_grid = grid;
      p.last_kernel = 4;
    } else {
      int S, grid, cg, cl;
      plan_tc(p, nq, a.KT, S, grid, cg, cl);
      P = S * ams::kEpiHalves;
      a.slots = (!a.gated && P >= a.k) ? 1 : 0;   // as launch_match_tc
      if (e0) AMS_CUDA_TRY(cudaEventRecord(e0, s));
      AMS_CUDA_TRY(ams::launch_match_tc(p, a, S, grid, cg, cl, sorted, s));
      if (e1) AMS_CUDA_TRY(cudaEventRecord(e1, s));
      p.last_splits = S;
      p.last_grid = grid;
      p.last_kernel = cl == 4 ? 5 : cg;
    }
    p.last_partials = P;
  }
  if (e0 && !(gate_first && p.cfg.dtype == AMS_DTYPE_BF16)) {
    if (p.local > 0) {
      p.ev_pending.emplace_back(e0, e1);
    } else {
      p.ev_free.push_back(e0);
      p.ev_free.push_back(e1);
    }
  }
  if (multi && p.peer_mode) {
    // fused NVLink exchange: merge + direct peer stores + flag completion, no NCCL launch
    ++p.epoch;
    const float* ps = p.part_s;
    const int32_t* pi = p.part_i;
    int32_t Pp = P, world_ids = p.cfg.world;
    int64_t Bids = p.B;
    if (gate_first && p.cfg.dtype == AMS_DTYPE_BF16) {   // shard lists already hold global ids
      AMS_CUDA_TRY(ams::launch_to_partials(shard_s, shard_i, nq, k, a.KT, p.part_s, p.part_i, s));
      Pp = 1;
      world_ids = 0;   // no shard map
      Bids = 0;
    }
    AMS_CUDA_TRY(ams::launch_exchange_push(a.KT, ps, pi, nq, Pp, k, p.peers, p.epoch, p.x_done, world_ids, Bids, s));
    AMS_CUDA_TRY(ams::launch_exchange_wait(a.KT, p.peers, nq, k, p.epoch, out_score, out_index, out_hit, threshold, s));
    p.launches += 2;
    return AMS_OK;
  }
  if (!(gate_first && p.cfg.dtype == AMS_DTYPE_BF16))
    AMS_CUDA_TRY(ams::launch_merge_partials(p, a, P, shard_s, shard_i, shard_hit,
                                            p.cfg.dtype == AMS_DTYPE_BF16 && p.local > 0, s));

  if (multi) {
    ncclComm_t comm = static_cast<ncclComm_t>(p.nccl_comm);
    const size_t cnt = (size_t)nq * k;
    if (ncclGroupStart() != ncclSuccess) return fail(pool, AMS_ERR_NCCL);
    if (ncclAllGather(p.shard_s, p.gath_s, cnt, ncclFloat32, comm, s) != ncclSuccess ||
        ncclAllGather(p.shard_i, p.gath_i, cnt, ncclInt64, comm, s) != ncclSuccess) {
      ncclGroupEnd();
      return fail(pool, AMS_ERR_NCCL);
    }
    if (ncclGroupEnd() != ncclSuccess) return fail(pool, AMS_ERR_NCCL);
    AMS_CUDA_TRY(ams::launch_merge_shards(p, a, p.cfg.world, k, p.gath_s, p.gath_i, out_score, out_index,
                                          out_hit, s));
  }
  return AMS_OK;
}

ams_status_t ams_match(ams_pool_t pool, const void* q_emb, const float* q_joints, int32_t nq, int32_t k,
                       float threshold, float gate_radius, int64_t* out_index, float* out_score,
                       uint8_t* out_hit, void* stream) {
  return match_impl(pool, q_emb, q_joints, nq, k, threshold, gate_radius, out_index, out_score, out_hit, stream,
                    false);
}

ams_status_t ams_match_gate_first(ams_pool_t pool, const void* q_emb, const float* q_joints, int32_t nq, int32_t k,
                                  float threshold, float gate_radius, int64_t* out_index, float* out_score,
                                  uint8_t* out_hit, void* stream) {
  return match_impl(pool, q_emb, q_joints, nq, k, threshold, gate_radius, out_index, out_score, out_hit, stream,
                    true);
}

ams_status_t ams_match_auto(ams_pool_t pool, const void* q_emb, const float* q_joints, int32_t nq, int32_t k,
                            float threshold, float gate_radius, int64_t* out_index, float* out_score, uint8_t* out_hit,
                            void* stream) {
  return match_impl(pool, q_emb, q_joints, nq, k, threshold, gate_radius, out_index, out_score, out_hit, stream,
                    false, true);
}

ams_status_t ams_pool_last_route(ams_pool_t pool, int32_t* route, double* est_eligible_per_query,
                                 double* est_ms_dense, double* est_ms_gate_first) {
  if (pool == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  const Pool& p = pool->p;
  if (route) *route = p.last_route;
  if (est_eligible_per_query) *est_eligible_per_query = p.est_valid ? p.est_elig : -1.0;
  if (est_ms_dense) *est_ms_dense = p.last_est_ms[0];
  if (est_ms_gate_first) *est_ms_gate_first = p.last_est_ms[1];
  return AMS_OK;
}

ams_status_t ams_merge_topk(const float* in_score, const int64_t* in_index, int32_t G, int32_t nq, int32_t kin,
                            int32_t k, float threshold, int64_t* out_index, float* out_score, uint8_t* out_hit,
                            void* stream) {
  ams_pool_s* pool = nullptr;
  if (in_score == nullptr || in_index == nullptr || out_index == nullptr || out_score == nullptr ||
      out_hit == nullptr || G < 1 || nq < 1 || kin < 1 || k < 1 || k > 64 || std::isnan(threshold))
    return AMS_ERR_INVALID_ARGUMENT;
  ams::MatchArgs a{};
  a.nq = nq;
  a.k = k;
  a.KT = ams::pick_KT(k);
  a.threshold = threshold;
  AMS_CUDA_TRY(ams::launch_merge_lists(a, G, kin, in_score, in_index, out_score, out_index, out_hit,
                                       static_cast<cudaStream_t>(stream)));
  return AMS_OK;
}

ams_status_t ams_pool_enable_peer_exchange(ams_pool_t pool) {
  if (pool == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  Pool& p = pool->p;
  if (pool_status(pool) != AMS_OK) return p.broken_st;
  const int G = p.cfg.world, r = p.cfg.rank;
  if (G < 1 || G > ams::kMaxPeers || p.nccl_comm == nullptr) return AMS_ERR_UNSUPPORTED;
  if (p.peer_mode) return AMS_OK;
  if (p.cfg.capacity >= ((int64_t)1 << 31)) return AMS_ERR_UNSUPPORTED;   // int32 ids in the partial lists
  AMS_CUDA_TRY(cudaSetDevice(p.cfg.device));
  ncclComm_t comm = static_cast<ncclComm_t>(p.nccl_comm);
  // Consensus protocol: every rank takes part in both all-gathers whatever its local
  // outcome, and every rank returns the same status (a rank that cannot allocate or map
  // must not leave its peers waiting inside a collective).
  //   block per rank = 3 IPC handles + int32 local status
  const size_t hb = 3 * sizeof(cudaIpcMemHandle_t) + sizeof(int32_t);
  std::vector<unsigned char> host((size_t)G * hb, 0);
  unsigned char* mine = host.data() + (size_t)r * hb;
  int32_t st_local = AMS_OK;
  const size_t slot = (size_t)2 * G * p.cfg.max_queries * p.cfg.max_k;
  bool ok = cudaMalloc((void**)&p.x_s, slot * 4) == cudaSuccess && cudaMalloc((void**)&p.x_i, slot * 8) == cudaSuccess &&
            cudaMalloc((void**)&p.x_flag, G * 8) == cudaSuccess && cudaMalloc((void**)&p.x_done, 4) == cudaSuccess &&
            cudaMalloc((void**)&p.x_barrier, (size_t)G * 4) == cudaSuccess;
  if (ok && p.x_err_host == nullptr)
    ok = cudaHostAlloc((void**)&p.x_err_host, sizeof(unsigned int), cudaHostAllocMapped) == cudaSuccess;
  unsigned int* err_dev = nullptr;
  if (ok) ok = cudaHostGetDevicePointer((void**)&err_dev, p.x_err_host, 0) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    st_local = AMS_ERR_OUT_OF_MEMORY;
  } else {
    *p.x_err_host = 0;
    if (cudaMemset(p.x_flag, 0, G * 8) != cudaSuccess || cudaMemset(p.x_done, 0, 4) != cudaSuccess ||
        cudaMemset(p.x_barrier, 0, (size_t)G * 4) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      cudaGetLastError();
      st_local = AMS_ERR_CUDA;
    }
  }
  cudaIpcMemHandle_t* h_mine = reinterpret_cast<cudaIpcMemHandle_t*>(mine);
  if (st_local == AMS_OK &&
      (cudaIpcGetMemHandle(&h_mine[0], p.x_s) != cudaSuccess || cudaIpcGetMemHandle(&h_mine[1], p.x_i) != cudaSuccess ||
       cudaIpcGetMemHandle(&h_mine[2], p.x_flag) != cudaSuccess)) {
    cudaGetLastError();
    st_local = AMS_ERR_UNSUPPORTED;
  }
  memcpy(mine + 3 * sizeof(cudaIpcMemHandle_t), &st_local, sizeof st_local);
  // all-gather 1: handles + local status
  void* dbuf = nullptr;
  AMS_CUDA_TRY(cudaMalloc(&dbuf, host.size()));
  AMS_CUDA_TRY(cudaMemcpy(static_cast<unsigned char*>(dbuf) + (size_t)r * hb, mine, hb, cudaMemcpyHostToDevice));
  if (ncclAllGather(static_cast<unsigned char*>(dbuf) + (size_t)r * hb, dbuf, hb, ncclChar, comm, nullptr) !=
      ncclSuccess) {
    cudaFree(dbuf);
    return fail(pool, AMS_ERR_NCCL);
  }
  AMS_CUDA_TRY(cudaDeviceSynchronize());
  AMS_CUDA_TRY(cudaMemcpy(host.data(), dbuf, host.size(), cudaMemcpyDeviceToHost));
  int32_t st_all = AMS_OK;
  for (int g = 0; g < G; ++g) {
    int32_t sg;
    memcpy(&sg, host.data() + (size_t)g * hb + 3 * sizeof(cudaIpcMemHandle_t), sizeof sg);
    if (sg != AMS_OK && st_all == AMS_OK) st_all = sg;
  }
  if (st_all != AMS_OK) {
    cudaFree(dbuf);
    free_peers(p);
    return static_cast<ams_status_t>(st_all == AMS_ERR_CUDA ? AMS_ERR_UNSUPPORTED : st_all);
  }
  ams::PeerTable pt{};
  pt.G = G;
  pt.rank = r;
  pt.max_q = p.cfg.max_queries;
  pt.max_k = p.cfg.max_k;
  pt.err = err_dev;
  pt.timeout_ns = ams::kPeerTimeoutNs;
  p.peer_mode = true;   // from here free_peers closes whatever was opened
  int32_t mapped = 1;
  for (int g = 0; g < G; ++g) {
    if (g == r) {
      pt.s[g] = p.x_s;
      pt.i[g] = p.x_i;
      pt.flag[g] = p.x_flag;
      continue;
    }
    const cudaIpcMemHandle_t* h = reinterpret_cast<const cudaIpcMemHandle_t*>(host.data() + (size_t)g * hb);
    void *a0 = nullptr, *a1 = nullptr, *a2 = nullptr;
    if (cudaIpcOpenMemHandle(&a0, h[0], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) pt.s[g] = static_cast<float*>(a0);
    if (cudaIpcOpenMemHandle(&a1, h[1], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) pt.i[g] = static_cast<int64_t*>(a1);
    if (cudaIpcOpenMemHandle(&a2, h[2], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess)
      pt.flag[g] = static_cast<unsigned long long*>(a2);
    if (!pt.s[g] || !pt.i[g] || !pt.flag[g]) {
      cudaGetLastError();
      mapped = 0;
    }
  }
  p.peers = pt;
  p.epoch = 0;
  // all-gather 2 (also the barrier: no rank writes into a peer before every rank has
  // mapped every peer): every rank's mapping outcome
  AMS_CUDA_TRY(cudaMemcpy(p.x_barrier + r, &mapped, 4, cudaMemcpyHostToDevice));
  if (ncclAllGather(p.x_barrier + r, p.x_barrier, 1, ncclUint32, comm, nullptr) != ncclSuccess) {
    cudaFree(dbuf);
    return fail(pool, AMS_ERR_NCCL);
  }
  AMS_CUDA_TRY(cudaDeviceSynchronize());
  cudaFree(dbuf);
  std::vector<uint32_t> all(G);
  AMS_CUDA_TRY(cudaMemcpy(all.data(), p.x_barrier, (size_t)G * 4, cudaMemcpyDeviceToHost));
  for (int g = 0; g < G; ++g)
    if (all[g] != 1) {
      free_peers(p);
      return AMS_ERR_UNSUPPORTED;
    }
  return AMS_OK;
}

ams_status_t ams_pool_status(ams_pool_t pool) {
  if (pool == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  return pool_status(pool);
}

ams_status_t ams_pool_size(ams_pool_t pool, int64_t* n) {
  if (pool == nullptr || n == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  *n = pool->p.size;
  return AMS_OK;
}

ams_status_t ams_pool_destroy(ams_pool_t pool) {
  if (pool == nullptr) return AMS_OK;
  Pool& p = pool->p;
  ams_status_t st = AMS_OK;
  cudaSetDevice(p.cfg.device);
  if (cudaDeviceSynchronize() != cudaSuccess) st = AMS_ERR_CUDA;
  if (p.nccl_comm != nullptr) {
    if (ncclCommDestroy(static_cast<ncclComm_t>(p.nccl_comm)) != ncclSuccess && st == AMS_OK) st = AMS_ERR_NCCL;
  }
  free_all(p);
  delete pool;
  return st;
}

ams_status_t ams_pool_set_profiling(ams_pool_t pool, int32_t enable) {
  if (pool == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  pool->p.profiling = enable != 0;
  return AMS_OK;
}

ams_status_t ams_pool_read_profile(ams_pool_t pool, double* kernel_ms, int64_t* kernel_launches) {
  if (pool == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  Pool& p = pool->p;
  double tot = 0.0;
  int64_t n = 0;
  for (auto& e : p.ev_pending) {
    if (cudaEventSynchronize(e.second) != cudaSuccess) return fail(pool, AMS_ERR_CUDA);
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, e.first, e.second) != cudaSuccess) return fail(pool, AMS_ERR_CUDA);
    tot += ms;
    ++n;
    p.ev_free.push_back(e.first);
    p.ev_free.push_back(e.second);
  }
  p.ev_pending.clear();
  if (kernel_ms) *kernel_ms = tot;
  if (kernel_launches) *kernel_launches = n;
  return AMS_OK;
}

ams_status_t ams_pool_launch_count(ams_pool_t pool, int64_t* launches) {
  if (pool == nullptr || launches == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  *launches = pool->p.launches;
  return AMS_OK;
}

ams_status_t ams_pool_set_kernel_policy(ams_pool_t pool, int32_t policy) {
  if (pool == nullptr || policy < 0 || policy > 15) return AMS_ERR_INVALID_ARGUMENT;
  pool->p.kernel_policy = policy;
  return AMS_OK;
}

ams_status_t ams_pool_last_plan(ams_pool_t pool, int32_t* splits, int32_t* partials, int32_t* grid,
                                int32_t* kernel_id) {
  if (pool == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  const Pool& p = pool->p;
  if (splits) *splits = p.last_splits;
  if (partials) *partials = p.last_partials;
  if (grid) *grid = p.last_grid;
  if (kernel_id) *kernel_id = p.last_kernel;
  return AMS_OK;
}

}  // extern "C"
