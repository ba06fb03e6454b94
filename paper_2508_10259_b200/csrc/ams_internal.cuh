// ams_internal.cuh -- pool state, shard map and kernel launchers shared by the
// C ABI (ams_capi.cu) and the kernels (ams_kernels.cu, ams_match_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

#include "../../include/ams.h"

namespace ams {

// --------------------------------------------------------------------------- tiling
constexpr int kBlockM = 128;     // queries per tcgen05 tile (TMEM lanes)
constexpr int kBlockN = 256;     // pool rows per tcgen05 tile (TMEM columns per buffer)
constexpr int kBlockK = 64;      // bf16 elements per stage row = one 128-B swizzle atom
constexpr int kRowAlign = 256;   // shard storage is padded to a multiple of this
constexpr int kEpiHalves = 2;    // epilogue warps per TMEM lane group (column halves)
constexpr int kSimtThreads = 128;
constexpr int kSnapBins = 65536;  // joint-0 bins of the gate-first index
constexpr int kQBins = 1024;      // joint-0 bins of a mid-size gate-first batch (query side)
constexpr int kGfRowsMaxQ = 16;   // gate-first batches up to this size: row kernel, unsorted
constexpr int kGfBinnedMaxQ = 1024;   // gated batches above kGfRowsMaxQ: joint-0 query bins; up to this
                                      // size their joints are staged in shared memory

// --------------------------------------------------------------------------- shard map
// Block-cyclic: global ordinal o -> block b = o / B, owner b % G, local (b / G) * B + o % B.
// The contiguous map is the special case B = ceil(capacity / G).
__host__ __device__ inline int64_t shard_block_size(int64_t capacity, int32_t world, int64_t block) {
  if (block > 0) return block;
  int64_t b = (capacity + world - 1) / world;
  return b > 0 ? b : 1;
}
__host__ __device__ inline int32_t shard_owner(int64_t o, int32_t world, int64_t B) {
  return static_cast<int32_t>((o / B) % world);
}
__host__ __device__ inline int64_t shard_local(int64_t o, int32_t world, int64_t B) {
  return (o / B / world) * B + o % B;
}
__host__ __device__ inline int64_t shard_global(int64_t l, int32_t rank, int32_t world, int64_t B) {
  return ((l / B) * world + rank) * B + l % B;
}
// rows of [0, n) owned by rank
__host__ __device__ inline int64_t shard_count(int64_t n, int32_t rank, int32_t world, int64_t B) {
  int64_t full = n / B, rem = n % B;
  int64_t blocks = full / world + ((full % world) > rank ? 1 : 0);
  return blocks * B + ((full % world) == rank ? rem : 0);
}

// Pool joints are stored tile-transposed: the JP joints of the 256 rows of tile T form a
// contiguous [JP][256] fp32 block, so one bulk copy stages a tile's joints and one
// 16-byte shared load yields joint t of four consecutive rows.
__host__ __device__ inline int64_t joint_offset(int64_t l, int t, int JP) {
  return ((l / kRowAlign) * JP + t) * kRowAlign + (l % kRowAlign);
}

// --------------------------------------------------------------------------- peer exchange
constexpr int kMaxPeers = 8;   // one NVSwitch box
// Receive buffers of every rank (local pointer for itself, CUDA-IPC mappings for peers):
// s/i are [2 parities][G senders][max_q][max_k]; flag is [G senders] epochs.
struct PeerTable {
  float* s[kMaxPeers];
  int64_t* i[kMaxPeers];
  unsigned long long* flag[kMaxPeers];
  int32_t G, rank;
  int32_t max_q, max_k;
  unsigned int* err;                // device alias of a host-mapped word: bit 0 = a wait timed out
  unsigned long long timeout_ns;    // bound on the consumer's flag wait
};
constexpr unsigned long long kPeerTimeoutNs = 10ull * 1000 * 1000 * 1000;   // 10 s

// --------------------------------------------------------------------------- pool
struct Pool {
  ams_pool_config_t cfg{};
  int32_t JP = 4;             // padded joint stride (4, 8 or 16)
  int64_t B = 1;              // shard block
  int64_t cap_shard = 0;      // rows this rank can hold
  int64_t cap_pad = 0;        // allocated rows (multiple of kRowAlign)
  int64_t size = 0;           // global rows appended
  int64_t local = 0;          // rows held by this rank
  int32_t num_sms = 148;
  int32_t max_clusters2 = 0;  // co-resident 2-CTA / 4-CTA clusters of the CTA-pair kernel
  int32_t max_clusters4 = 0;
  int32_t KT_max = 8;
  bool broken = false;
  ams_status_t broken_st = AMS_OK;   // status every call returns once broken
  bool collective = false;    // world > 1, or world == 1 with an nccl_id: shard lists go
                              // through the NCCL all-gather + shard merge (or peer exchange)

  // shard storage
  void* emb = nullptr;        // [cap_pad, d] bf16 or fp32
  float* inv_norm = nullptr;  // [cap_pad]
  float* joints = nullptr;    // [cap_pad / 256][JP][256] (joint_offset)

  // query workspace
  int32_t q_pad = 0;          // max_queries rounded up to kBlockM
  void* q_stage = nullptr;    // [q_pad, d]
  float* q_inv = nullptr;     // [q_pad]
  float* q_joints = nullptr;  // [q_pad, JP]
  // host-sourced queries: double-buffered staging filled on copy_stream, so the H2D of
  // call i+1 overlaps the kernels of call i (staged[b] / consumed[b] order the reuse)
  float* q_joints_raw[2] = {nullptr, nullptr};  // [max_queries, J]
  void* q_raw[2] = {nullptr, nullptr};          // [max_queries, d], gathered into q_stage
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t staged[2] = {nullptr, nullptr};
  cudaEvent_t consumed[2] = {nullptr, nullptr};
  int32_t stage_buf = 0;
  int32_t* q_perm = nullptr;  // [q_pad] staged position -> caller's query (joint-0 order)

  // partial top-k lists [nq][P][KT]
  int64_t part_cap = 0;       // entries
  float* part_s = nullptr;
  int32_t* part_i = nullptr;
  int32_t P_max = 0;

  // shard top-k and the all-gathered lists
  float* shard_s = nullptr;      // [max_q, max_k]
  int64_t* shard_i = nullptr;
  float* gath_s = nullptr;       // [world, max_q, max_k]
  int64_t* gath_i = nullptr;

  // append staging (host sources)
  int64_t stage_rows = 0;
  void* stage_emb = nullptr;
  float* stage_joints = nullptr;

  // small-batch kernel on CTA pairs: per (CTA, epilogue warp) list workspace,
  // [num_sms][4 warps][8 slots][8 entries][32 lanes] scores and local rows
  float* scan_glist_s = nullptr;
  int32_t* scan_glist_i = nullptr;
  uint32_t* bound = nullptr;  // [q_pad] per-query admission lower bound (tcgen05 path)
  uint32_t* slots = nullptr;  // [q_pad][KT_max] union-bound slots (tcgen05 path, ungated)

  // gate-first variant: per-query candidate buckets
  int32_t gf_cap = 0;
  uint32_t* gf_cnt = nullptr;  // [q_pad]
  int32_t* gf_cand = nullptr;  // [q_pad, gf_cap] local rows
  int32_t* gf_qbins = nullptr; // [kQBins + 1] staged-query offsets of the joint-0 query bins, then {lo, scale}
  // per-device launch facts of the gate-first kernels, cached on the pool (one device)
  size_t gf_rows_smem_opt = 0;  // dynamic shared memory opted in for the binned row kernels
  int gf_occ[3][4] = {};        // resident gate_scan blocks per SM, [JP 4/8/16][QT 32/64/128/256]
  // gate-first joint-0 index (built lazily by the first sorted gate-first call): local rows
  // [0, snap_L) bucket-sorted by joint 0 into kSnapBins linear bins; rows appended since
  // are scanned in plain order until the next rebuild
  int64_t snap_L = 0;
  float* snap_j = nullptr;      // [cap_pad/256][JP][256] joints in snapshot order
  int32_t* snap_id = nullptr;   // [cap_pad] snapshot position -> local row
  int32_t* snap_off = nullptr;  // [kSnapBins + 1] first snapshot position of each bin
  uint32_t* snap_aux = nullptr; // [kSnapBins] histogram / cursor, then {min, max} (ordered u32), {lo, scale}

  CUtensorMap tmap_pool{};   // bf16 pool [cap_pad, d], box {64, 256}, SW128 (CTA tile)
  CUtensorMap tmap_pool2{};  // bf16 pool [cap_pad, d], box {64, 128}, SW128 (CTA-pair half tile)
  CUtensorMap tmap_pool4{};  // bf16 pool [cap_pad, d], box {64, 64}, SW128 (multicast quarter tile)
  CUtensorMap tmap_q{};      // bf16 queries [q_pad, d], box {64, 128}, SW128
  CUtensorMap tmap_qs[16]{}; // bf16 queries [q_pad, d], box {64, 8 (i + 1)}, SW128 (small-batch kernel)
  size_t simt_smem_opt[4] = {0, 0, 0, 0};   // dynamic smem opted in per SIMT kernel (KT 8/16/32/64)
  int32_t kernel_policy = 0; // bit 0: never the small-batch kernel; bit 1: 4-CTA multicast clusters;
                             // bit 2: wide (two tiles per stage) small-batch CTA pairs;
                             // bit 3: ungated 129-256-query batches on the small-batch CTA pairs

  void* nccl_comm = nullptr;  // ncclComm_t

  // fused NVLink exchange (opt-in, ams_pool_enable_peer_exchange)
  bool peer_mode = false;
  PeerTable peers{};
  unsigned long long epoch = 0;
  unsigned int* x_done = nullptr;       // [1] arrival counter of merge_push_kernel's blocks
  unsigned int* x_barrier = nullptr;    // [world] scratch of the mapping barrier all-gather
  unsigned int* x_err_host = nullptr;   // host-mapped error word (PeerTable::err aliases it)
  float* x_s = nullptr;                 // own receive buffers (also peers.s[rank])
  int64_t* x_i = nullptr;
  unsigned long long* x_flag = nullptr;

  // ams_match_auto: cached estimate of eligible rows per query (refreshed asynchronously)
  unsigned long long* est_dev = nullptr;     // [1] sampled eligible pairs
  unsigned long long* est_host = nullptr;    // pinned copy of est_dev
  cudaEvent_t est_ready = nullptr;           // recorded after the D2H of a refresh
  bool est_pending = false, est_valid = false;
  float est_g2 = 0.0f;                       // gate of the cached estimate
  int64_t est_L = 0;                         // local rows when it was taken
  int32_t est_rows = 0, est_queries = 0;     // sample sizes of the pending / adopted refresh
  double est_elig = 0.0;                     // eligible rows per query (local shard)
  int64_t est_calls = 0;
  int32_t last_route = -1;                   // 0 dense, 1 gate-first
  double last_est_ms[2] = {0.0, 0.0};        // cost model of the last auto call (dense, gate-first)

  // instrumentation
  bool profiling = false;
  std::vector<cudaEvent_t> ev_free;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending;
  int64_t launches = 0;
  int32_t last_splits = 0, last_partials = 0, last_grid = 0, last_kernel = -1;
};

// --------------------------------------------------------------------------- launchers
// All return cudaError_t of the launch; `launches` is incremented per kernel launched.
// Launch configuration of a programmatic dependent launch: the kernel may start while
// the previous kernel on `s` is still running and must call ptx::griddep_wait() before it
// reads that kernel's results (ams.h: "programmatic dependents").  attr: caller storage.
inline cudaLaunchConfig_t pdl_config(dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                     cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

struct MatchArgs {
  int32_t nq, k, KT;
  float g2;           // fp32(gate_radius^2); +inf disables the gate
  int32_t gated;      // g2 < +inf
  float threshold;
  int32_t slots;      // the tcgen05 kernel filled p.slots (union bound) for the merge
  int32_t zeroed;     // query prep already zeroed this call's counters (p.bound / p.slots or p.gf_cnt)
  int32_t qbins;      // gate-first: queries staged in joint-0 bin order (launch_query_order_j0)
};

cudaError_t launch_append(Pool& p, const void* emb_src, const float* joints_src, int64_t n_src,
                          int64_t first_global, cudaStream_t s);
// perm (device, may be null = identity): staged row q is the caller's query perm[q].
// Also zeroes zero_a[0, n_zero_a) and zero_b[0, n_zero_b): the counters of the kernel that
// follows (dense: p.bound and p.slots; gate-first: p.gf_cnt), which its launcher then no
// longer memsets (MatchArgs::zeroed), so that kernel can be the prep's programmatic dependent.
cudaError_t launch_query_prep(Pool& p, const void* q_src, const float* qj_src, int32_t nq, const int32_t* perm,
                              uint32_t* zero_a, int32_t n_zero_a, uint32_t* zero_b, int32_t n_zero_b,
                              cudaStream_t s);
// p.q_perm <- the queries ordered by joint 0 (counting sort into linear bins; one block)
cudaError_t launch_query_order(Pool& p, const float* qj_src, int32_t nq, cudaStream_t s);
cudaError_t launch_match_simt(Pool& p, const MatchArgs& a, int32_t splits, cudaStream_t s);
// fp32 exact, ungated calls: tiles of 32 rows x 16 queries, one partial list per (query,
// row tile); f32_tile_lists(L) = the number of lists per query
int f32_tile_lists(int64_t L);
cudaError_t launch_match_f32_tile(Pool& p, const MatchArgs& a, cudaStream_t s);
// cg = 1: one CTA per 128x256 tile; cg = 2: CTA pair (cta_group::2) per 256x256 tile
// sorted: queries were staged through p.q_perm (partials land at the caller's query index)
// cl: CTAs per cluster (cg, or 4 for cg = 2: two CTA pairs sharing multicast pool rows;
// needs an even number of 256-query tiles)
cudaError_t launch_match_tc(Pool& p, const MatchArgs& a, int32_t splits, int32_t grid, int32_t cg, int32_t cl,
                            bool sorted, cudaStream_t s);
int tc_query_tile(int cg);
int tc_max_active_clusters(int cl);   // co-resident clusters of cl CTAs (CTA-pair kernel); 0 on error
// small-batch kernel (pool rows on the MMA M side, queries on N): pipeline stages that fit
// shared memory for this batch, 0 if the batch is not eligible (nq > 256, KT > 32, KT != 8
// above 128 queries, or the per-lane register lists would not fit)
int scan_stages(const Pool& p, int nq, int KT);
int scan_cg(int nq);                 // CTAs per tile: 1 (nq <= 128) or 2 (CTA pair)
int scan_w(const Pool& p, int nq, int KT);   // tiles per pipeline stage (2: wide CTA pair)
int scan_lists_per_split(int nq, int KT, bool gated);   // partial lists per row split (1: warps merged in the CTA)
cudaError_t launch_match_scan(Pool& p, const MatchArgs& a, int32_t splits, int32_t grid, cudaStream_t s);
// merge [nq][P][KT] local lists -> [nq][k] (fp32, global int64); writes hit if out_hit != null
// tc_bounds: the lists come from launch_match_tc, whose per-query lower bounds (p.bound,
// p.slots) prune entries that cannot reach the top k
cudaError_t launch_merge_partials(Pool& p, const MatchArgs& a, int32_t P, float* out_s, int64_t* out_i,
                                  uint8_t* out_hit, bool tc_bounds, cudaStream_t s);
// merge [G][nq][kin] global lists -> [nq][k] + hit
cudaError_t launch_merge_shards(Pool& p, const MatchArgs& a, int32_t G, int32_t kin, const float* in_s,
                                const int64_t* in_i, float* out_s, int64_t* out_i, uint8_t* out_hit,
                                cudaStream_t s);

cudaError_t launch_merge_lists(const MatchArgs& a, int32_t G, int32_t kin, const float* in_s, const int64_t* in_i,
                               float* out_s, int64_t* out_i, uint8_t* out_hit, cudaStream_t s);
// gate-first sparse variant (bf16 pools): writes [nq][k] (+hit if out_hit)
// sorted: queries were staged through p.q_perm (outputs land at the caller's query index)
cudaError_t launch_gate_first(Pool& p, const MatchArgs& a, float* out_s, int64_t* out_i, uint8_t* out_hit,
                              bool sorted, cudaStream_t s);
// p.q_perm <- the queries in kQBins linear joint-0 bins (one block),
// p.gf_qbins <- the bins' staged offsets and {lo, scale}: the gate-first row kernel then
// visits, per pool row, only the queries of the bins within gamma of its joint 0
cudaError_t launch_query_order_j0(Pool& p, const float* qj_src, int32_t nq, cudaStream_t s);
cudaError_t launch_exchange_push(int KT, const float* ps, const int32_t* pi, int32_t nq, int32_t P, int32_t k,
                                 const PeerTable& pt, unsigned long long epoch, unsigned int* done, int32_t world_ids,
                                 int64_t B, cudaStream_t s);
cudaError_t launch_exchange_wait(int KT, const PeerTable& pt, int32_t nq, int32_t k, unsigned long long epoch,
                                 float* os, int64_t* oi, uint8_t* oh, float th, cudaStream_t s);
cudaError_t launch_to_partials(const float* s, const int64_t* i, int32_t nq, int32_t k, int32_t KT, float* ps,
                               int32_t* pi, cudaStream_t st);
int pick_KT(int k);
// ams_match_auto's pass-rate estimate: out[0] = eligible pairs among a strided sample of
// <= kEstQueries of the caller's raw query joints [nq][J] x <= kEstRows local rows
constexpr int kEstQueries = 64;
constexpr int64_t kEstRows = 32768;
cudaError_t launch_gate_estimate(Pool& p, const float* qj_raw, int32_t nq, float g2, unsigned long long* out,
                                 int32_t* rows_sampled, int32_t* queries_sampled, cudaStream_t s);

}  // namespace ams
