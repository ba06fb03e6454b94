/*
 * ams.h -- C ABI of the B200-native action-context matcher (AMS, arXiv 2508.10259).
 *
 * The hot path this library implements is the action-context pool lookup of AMS:
 *   PAPER.md:486 (3.2.1)   a context holds "data from the robot's joints and the output
 *                           embedding obtained from the final inference";
 *   PAPER.md:489 (3.2.1)   "During each inference, the system first checks the action
 *                           context pool to see if any similar and reusable intermediate
 *                           states exist";
 *   PAPER.md:494 (3.2.1)   "After one single inference, AMS adds the unseen vector ... into
 *                           the context pool" (-> ams_pool_append);
 *   PAPER.md:865 (4)       replay retrieves "stored contexts from the context pool one by
 *                           one" (-> the ranked top-k list);
 *   SPEC.md:186-190        lookup: best match "or none below threshold";
 *   BASELINE.json north_star: cosine similarity over the embedding, gated by the L2
 *                           distance between joint states, per-query top-k, a cosine
 *                           threshold giving the replay hit/miss flag, ties to the
 *                           lowest index; ams_pool_create / ams_pool_append /
 *                           ams_match / ams_pool_destroy.
 * The exact definition (and every reading where the paper is silent) is in DESIGN.md
 * "Method" / "Readings"; the CPU oracle in oracle/ computes the same definition.
 *
 * Conventions (all entry points):
 *   - Every call returns ams_status_t and never throws or aborts.
 *   - The library owns pool storage and all workspace; the caller owns every buffer it
 *     passes.  Input buffers may be host or device pointers (detected through UVA);
 *     output buffers of ams_match must be DEVICE pointers.
 *   - Work is enqueued on the caller's stream `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream); calls return after enqueue.  Inputs must stay
 *     valid until the stream reaches that point.  An append is visible to every later
 *     match on the same stream.  Inside a call, the kernels after the first are launched
 *     as programmatic dependents of their predecessor (they start early and wait on the
 *     device for its results); the call's first kernel is an ordinary launch, so it
 *     waits for all earlier work on `stream`, and so does the caller's next ordinary
 *     launch for the whole call.
 *   - A pool is NOT thread-safe; callers serialise calls on one pool ("a
 *     single pool serializes writers").  Calls on one pool share its device workspace
 *     (staging, partial lists), so they must also be ordered on the device: issue them on
 *     one stream, or order the streams (events) between calls.
 *   - Argument errors are detected synchronously and nothing is enqueued.
 *   - After AMS_ERR_CUDA / AMS_ERR_NCCL the pool is unusable and must be destroyed.
 *   - Multi-GPU (world > 1): one process per GPU; create / append / match / destroy are
 *     collective (every rank calls them in the same order with identical arguments).
 *   - CUDA graphs: ams_match / ams_match_gate_first with DEVICE inputs on a pool without
 *     the peer exchange are stream-ordered with no host synchronisation and may be
 *     captured; the plan (kernel, splits) is frozen at capture, so re-capture after
 *     appends.  During capture, host-resident inputs (a pageable copy) and peer-exchange
 *     pools (a host epoch counter) return AMS_ERR_UNSUPPORTED and the pool stays usable;
 *     the same holds for ams_pool_append with host-resident rows.
 */
#ifndef AMS_H_
#define AMS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMS_ABI_VERSION 2

typedef struct ams_pool_s* ams_pool_t; /* opaque, library-owned */

typedef enum {
  AMS_OK = 0,
  AMS_ERR_INVALID_ARGUMENT = 1,
  AMS_ERR_CAPACITY = 2,      /* SPEC.md:181 CapacityError: append would exceed capacity */
  AMS_ERR_OUT_OF_MEMORY = 3,
  AMS_ERR_CUDA = 4,          /* sticky device error; destroy the pool */
  AMS_ERR_NCCL = 5,          /* collective failure; destroy the pool */
  AMS_ERR_UNSUPPORTED = 6,   /* e.g. no sm_100 device, d not a multiple of 64 */
  AMS_ERR_INTERNAL = 7
} ams_status_t;

typedef enum { AMS_DTYPE_BF16 = 0, AMS_DTYPE_FP32 = 1 } ams_dtype_t;

typedef struct {
  int32_t dim;            /* d, embedding width; multiple of 64, 64 <= d <= 16384 */
  int32_t joint_dim;      /* J in [1, 16] joint DoF (7-DoF output action) */
  ams_dtype_t dtype;      /* storage type of pool AND query embeddings (reading R10).
                             BF16: tensor-core path, fp32 accumulate (tolerance 2e-3);
                             FP32: canonical-order path, bit-exact vs the oracle */
  int64_t capacity;       /* max global rows; storage is preallocated at create */
  int32_t max_queries;    /* >= every nq passed to ams_match (workspace sizing) */
  int32_t max_k;          /* >= every k passed to ams_match; 1 <= max_k <= 64 */
  int32_t device;         /* CUDA ordinal used by this rank */
  int32_t rank, world;    /* world == 1: single GPU, no NCCL; world <= 64 */
  const void* nccl_id;    /* 128-byte ncclUniqueId, identical on all ranks; NULL if world == 1.
                             world == 1 with a non-NULL id builds a 1-rank communicator and
                             runs the world > 1 path (shard merge, NCCL all-gather, final
                             merge; peer exchange if enabled) on one GPU -- results are
                             identical; used by the tests to exercise that path */
  int64_t shard_block;    /* rows per block of the block-cyclic row map (global append
                             ordinal o lives on rank (o / B) % world);
                             0 -> contiguous: B = ceil(capacity / world) */
} ams_pool_config_t;

/* Writes a fresh 128-byte NCCL unique id to out128 (rank 0 calls it; the harness
 * broadcasts the bytes to the other ranks, e.g. through torch.distributed). */
ams_status_t ams_get_nccl_unique_id(void* out128);

/* Creates a pool on cfg->device: allocates the rank's shard (bf16 or fp32 embeddings
 * [cap_shard, d] row-major, fp32 inverse norms [cap_shard], fp32 joints [cap_shard, JP]
 * with JP = J rounded up to 4, 8 or 16 and zero padding) plus every workspace
 * ams_match needs (ams_match never allocates).  Collective over NCCL if world > 1.
 * Errors: AMS_ERR_INVALID_ARGUMENT (null pointers, bad sizes), AMS_ERR_UNSUPPORTED
 * (device is not sm_100), AMS_ERR_OUT_OF_MEMORY, AMS_ERR_CUDA, AMS_ERR_NCCL. */
ams_status_t ams_pool_create(const ams_pool_config_t* cfg, ams_pool_t* out);

/* Record: appends n contexts.  emb is [n, d] (bf16 bits as uint16, or
 * fp32, per cfg.dtype) row-major, joints is [n, J] fp32 row-major; host or device.
 * Rows receive the global append ordinals [size, size + n); *first_index (host, may
 * be NULL) receives `size`.  Each rank keeps the rows its shard map owns and computes
 * their inverse L2 norms from the STORED values (bf16: fp64 sum, rounded once to fp32;
 * fp32: canonical in-order fmaf chain, IEEE sqrt and division).  With DEVICE buffers
 * only the rows this rank owns are read (a rank that owns none of [size, size + n) may
 * pass any valid device pointer); host buffers are staged in full.
 * Errors: AMS_ERR_INVALID_ARGUMENT (null pool, n < 0, null data with n > 0),
 * AMS_ERR_CAPACITY (size + n > capacity; nothing is appended), AMS_ERR_CUDA. */
ams_status_t ams_pool_append(ams_pool_t pool, const void* emb, const float* joints, int64_t n,
                             int64_t* first_index, void* stream);

/* Lookup: for each of nq queries (q_emb [nq, d] in the
 * pool dtype, q_joints [nq, J] fp32; host or device):
 *   score(i, j)  = (dot(q_i, e_j) * inv_q_i) * inv_e_j                    (cosine)
 *   eligible(i,j) = sum_t (r_it - p_jt)^2 <= fp32(gate_radius^2), canonical fp32
 *                   (the joint gate; gate_radius = +inf disables it)
 *   out_index[i, 0..k)  global append ordinals of the k best eligible rows ordered by
 *                       (score desc, index asc); -1 padding when fewer are eligible
 *   out_score[i, 0..k)  their fp32 scores; -inf padding
 *   out_hit[i]          1 iff out_index[i,0] >= 0 and out_score[i,0] >= threshold
 * Outputs are DEVICE buffers: out_index int64 [nq, k], out_score fp32 [nq, k],
 * out_hit uint8 [nq].  With world > 1 every rank receives identical outputs.
 * Host-resident q_emb / q_joints are copied on a pool-internal copy stream into one of
 * two staging buffers and `stream` waits for that copy only, so the H2D of one call
 * overlaps the kernels still running from the previous call on `stream`; the host
 * buffers must stay valid (and unmodified) until `stream` reaches this call.
 * Errors: AMS_ERR_INVALID_ARGUMENT (null pool/pointers, nq < 1 or > max_queries,
 * k < 1 or > max_k, NaN threshold, NaN or negative gate_radius), AMS_ERR_CUDA,
 * AMS_ERR_NCCL.  k larger than the pool is legal (padded). */
ams_status_t ams_match(ams_pool_t pool, const void* q_emb, const float* q_joints, int32_t nq,
                       int32_t k, float threshold, float gate_radius, int64_t* out_index,
                       float* out_score, uint8_t* out_hit, void* stream);

/* Gate-first sparse variant of ams_match: identical arguments,
 * semantics, outputs and errors.  It evaluates the canonical joint gate for every
 * (query, row) pair first -- reading only the pool's joints -- and computes cosine scores
 * only for eligible pairs (CUDA-core dot products; the scores may differ from ams_match's
 * tensor-core accumulation in the last fp32 bits, both within the stated tolerance).
 * Efficient when the gate is selective (few eligible rows per query); with a wide gate
 * it stays exact but degrades to a per-query scan on the GPU.  fp32 pools use the exact
 * path of ams_match, which already evaluates the gate first.
 * On pools of >= 64 K local rows, batches of >= 129 queries use a joint-0 index of the
 * pool (rows bucket-sorted by joint 0; built on first use -- allocating cap * (4 * JP + 4)
 * bytes, JP = J rounded up to 4/8/16 -- and rebuilt once more than max(64 K, L/32) rows
 * were appended since): each block of queries scans only the rows whose joint 0 lies
 * within gamma of its queries' joint 0.  Results are unchanged. */
ams_status_t ams_match_gate_first(ams_pool_t pool, const void* q_emb, const float* q_joints, int32_t nq,
                                  int32_t k, float threshold, float gate_radius, int64_t* out_index,
                                  float* out_score, uint8_t* out_hit, void* stream);

/* Route-selecting variant of ams_match ("select by measured
 * pass-rate"): identical arguments, semantics, outputs and errors; the pool picks the
 * dense tensor-core path (ams_match) or the gate-first path (ams_match_gate_first) for
 * this call from a cost model fed by an estimate of the eligible rows per query -- the
 * exact canonical gate over a strided sample of <= 64 of the call's queries x <= 32768
 * local rows.  The estimate is taken synchronously (stream synchronised once) on the
 * first gated call, when the gate radius changes or the shard size changed 2x, and
 * refreshed asynchronously every 64 calls otherwise.  Ungated calls and fp32 pools always
 * take the dense/exact path.  Both routes are exact; scores may differ between routes in
 * the last fp32 bits (tensor-core vs CUDA-core accumulation), within the stated
 * tolerance.  With world > 1 each rank chooses for its own shard.  Not capturable in a
 * CUDA graph (AMS_ERR_UNSUPPORTED during capture).  The route of the last call:
 * ams_pool_last_route. */
ams_status_t ams_match_auto(ams_pool_t pool, const void* q_emb, const float* q_joints, int32_t nq,
                            int32_t k, float threshold, float gate_radius, int64_t* out_index,
                            float* out_score, uint8_t* out_hit, void* stream);

/* Route of the last ams_match_auto call on this pool: *route 0 = dense, 1 = gate-first,
 * -1 = none yet; the estimated eligible rows per query of the local shard (-1 if none),
 * and the cost model's estimates in ms for both routes (0 if the route was forced by an
 * ungated call or an fp32 pool).  Any output pointer may be NULL.
 * Errors: AMS_ERR_INVALID_ARGUMENT (null pool). */
ams_status_t ams_pool_last_route(ams_pool_t pool, int32_t* route, double* est_eligible_per_query,
                                 double* est_ms_dense, double* est_ms_gate_first);

/* The final k-way merge (north_star "a final k-way merge kernel"; step a7 of
 * DESIGN.md): merges G ranked lists per query -- in_score/in_index are DEVICE arrays
 * [G, nq, kin] (fp32 score, int64 global index, -1 padding), each list ordered by
 * (score desc, index asc) -- into out_index/out_score [nq, k] and out_hit [nq] (device)
 * with the same ordering, padding and hit rule as ams_match.  ams_match uses the same
 * kernel after its NCCL all-gather; this entry serves callers that shard themselves.
 * Errors: AMS_ERR_INVALID_ARGUMENT (null pointers, G < 1, nq < 1, kin < 1, k < 1,
 * k > 64, NaN threshold), AMS_ERR_CUDA. */
ams_status_t ams_merge_topk(const float* in_score, const int64_t* in_index, int32_t G, int32_t nq,
                            int32_t kin, int32_t k, float threshold, int64_t* out_index,
                            float* out_score, uint8_t* out_hit, void* stream);

/* ---- fused NVLink shard exchange (opt-in) ----
 * Replaces, for this pool, the NCCL all-gather + merge of ams_match / ams_match_gate_first
 * at world > 1 (north_star "row-sharded ... with an NCCL all-gather plus a final k-way
 * merge"; PAPER.md:486-489 define the lookup itself) by direct peer stores: each rank's
 * intra-GPU merge kernel writes its [nq, k] list into a receive slot of EVERY rank's
 * buffer over NVLink (CUDA IPC mappings), then raises an epoch flag with a system-scope
 * release; the final merge kernel acquires all G flags and merges.  Outputs are identical
 * to the NCCL path.  Collective: every rank calls it once after ams_pool_create (the
 * three IPC handles per rank travel over the pool's NCCL communicator).  Requires all
 * ranks on one node with peer access; the pool's matches must be issued by every rank in
 * the same order (as with the NCCL path).  The final merge waits for each peer's flag to
 * reach the call's epoch for at most 10 s (device globaltimer); on timeout it writes
 * padding (-1, -inf, miss), records the failure in a host-mapped error word, and the
 * pool's next call (or ams_pool_status) returns AMS_ERR_NCCL -- a dead or desynchronised
 * peer cannot hang the GPU.  Not capturable in a CUDA graph (the epoch is a host counter;
 * ams_match returns AMS_ERR_UNSUPPORTED during capture).  Errors: AMS_ERR_INVALID_ARGUMENT (null pool),
 * AMS_ERR_UNSUPPORTED (pool without a communicator -- world == 1 and no nccl_id --,
 * world > 8, capacity >= 2^31, IPC unavailable),
 * AMS_ERR_OUT_OF_MEMORY, AMS_ERR_NCCL, AMS_ERR_CUDA.  Idempotent. */
ams_status_t ams_pool_enable_peer_exchange(ams_pool_t pool);

/* Single-device self-test of the exchange kernels: G (1..8) virtual ranks, each with its
 * own receive buffer and flag array on the current device, run `rounds` exchanges
 * (epochs 1..rounds, alternating buffer parity).  in_score/in_index: DEVICE
 * [rounds][G][nq][k] ranked lists (score desc, index asc; -inf / -1 padding; ids < 2^31);
 * out_score/out_index: DEVICE [rounds][G][nq][k]; out_hit [rounds][G][nq] -- virtual rank
 * g's merged result of round r, which must equal ams_merge_topk of that round's G lists
 * for every g.  Every consumer launch is enqueued on `stream` after the producer launches
 * it waits for, so no kernel waits on a concurrently running kernel.  flags:
 *   AMS_SELFTEST_LATE_CONSUMER  virtual rank G-1 consumes round r-1 only after the other
 *                               ranks produced round r (their flags are ahead of the epoch
 *                               it waits for; G >= 2); results must be unchanged;
 *   AMS_SELFTEST_DROP_LAST      virtual rank G-1 never produces the last round: the other
 *                               ranks' waits time out after 20 ms, their outputs of that
 *                               round are padding, and the call returns AMS_ERR_NCCL.
 * Allocates and frees its own buffers; synchronises `stream`.  Errors:
 * AMS_ERR_INVALID_ARGUMENT (G, nq, k (1..64), rounds or flags out of range, null
 * pointers), AMS_ERR_OUT_OF_MEMORY, AMS_ERR_CUDA, AMS_ERR_NCCL (a wait timed out). */
#define AMS_SELFTEST_LATE_CONSUMER 1
#define AMS_SELFTEST_DROP_LAST 2
ams_status_t ams_exchange_selftest(int32_t G, int32_t nq, int32_t k, int32_t rounds, float threshold,
                                   const float* in_score, const int64_t* in_index, float* out_score,
                                   int64_t* out_index, uint8_t* out_hit, int32_t flags, void* stream);

/* Sticky status of a pool without synchronising: AMS_ERR_NCCL once a peer-exchange wait
 * timed out (visible as soon as the timed-out kernel wrote it; synchronise the stream
 * first for a definite answer), AMS_ERR_CUDA after an earlier CUDA failure, else AMS_OK.
 * Errors: AMS_ERR_INVALID_ARGUMENT (null pool). */
ams_status_t ams_pool_status(ams_pool_t pool);

/* Identity of this build of the library: a hash of the sources, headers and compile flags
 * it was built from (static string, never NULL; "unknown" if built without it).  Profiles
 * record it so a reported DRAM-traffic figure can be tied to the code it measured. */
const char* ams_build_id(void);

/* ---- two-phase action hash (Algorithm 1) ----
 * Phase 1 hashes every s-byte segment of every input independently, phase 2 folds an
 * input's segment hashes ("modular calculation").
 * Concretisation: h_i = polynomial hash of segment i's bytes,
 * h = (h*257 + byte) mod (2^61 - 1) from 0; H_final = fold (acc*257 + h_i) mod
 * (2^61 - 1) from 0; an empty input hashes to 0.  Bit-exact; the result is the
 * "unique index for action lookup and management" of PAPER.md:541. */
typedef struct ams_hasher_s* ams_hasher_t;

/* Preallocates a hasher on `device` for up to max_inputs inputs and max_bytes input
 * bytes per call (host-resident inputs are staged into a device buffer of that size;
 * device-resident inputs are read in place); segment_size = s (1..2^24; SPEC default
 * 4096).  Errors: AMS_ERR_INVALID_ARGUMENT,
 * AMS_ERR_OUT_OF_MEMORY, AMS_ERR_CUDA. */
ams_status_t ams_hasher_create(int32_t device, int64_t max_inputs, int64_t max_bytes, int64_t segment_size,
                               ams_hasher_t* out);

/* Hashes n_inputs byte strings: input i is data[offsets[i], offsets[i+1]) (CSR).  `data`
 * is host or device memory; `offsets` is a HOST array of n_inputs + 1 non-decreasing
 * int64 values (read synchronously); out_hash is a DEVICE array of n_inputs uint64.
 * Enqueued on `stream`; a later call waits for the previous call's staging to drain.
 * Errors: AMS_ERR_INVALID_ARGUMENT (null pointers, n_inputs out of range, decreasing
 * offsets), AMS_ERR_CAPACITY (more than max_bytes input bytes),
 * AMS_ERR_CUDA. */
ams_status_t ams_hash_actions(ams_hasher_t hasher, const uint8_t* data, const int64_t* offsets,
                              int32_t n_inputs, uint64_t* out_hash, void* stream);

/* Segments of the last ams_hash_actions call, and how many of them phase 1 hashed on the
 * tensor cores: full segments starting 16-B aligned, when s is a multiple of 128 and
 * <= 8192 -- each segment hash is then an exact u8 x u8 -> s32 contraction of its bytes
 * with the 8-bit limbs of the weights B^(s-1-k) mod M (tcgen05.mma kind::i8), folded mod
 * M.  All other segments use the CUDA-core path; the results are identical.
 * Errors: AMS_ERR_INVALID_ARGUMENT (null hasher). */
ams_status_t ams_hasher_last_stats(ams_hasher_t hasher, int64_t* segments, int64_t* tc_segments);

/* Synchronises the device and frees the hasher.  NULL is a no-op. */
ams_status_t ams_hasher_destroy(ams_hasher_t hasher);

/* ---- virtual-action store ----
 * "uniquely numbered actions with independent reference counts ... stored in a
 * contiguous area ... Any action whose reference count drops to zero is removed."
 * Ids are the two-phase hashes H_final (ams_hash_actions).  Device hash table + an
 * append-only device byte arena; every operation is batched and stream-ordered. */
typedef struct ams_vstore_s* ams_vstore_t;

/* Per-action status written by ams_vstore_intern. */
#define AMS_VSTORE_NEW 0        /* entry created, refcount 1, bytes copied to the arena */
#define AMS_VSTORE_DEDUP 1      /* identical bytes already stored: refcount incremented */
#define AMS_VSTORE_COLLISION 2  /* id present with DIFFERENT bytes: nothing changed (SPEC CollisionError) */
#define AMS_VSTORE_FULL 3       /* table or arena full: nothing stored */

/* max_actions live entries (table capacity 2x, power of two), arena_bytes of action
 * bytes, batches of up to max_batch actions / max_batch_bytes bytes. */
ams_status_t ams_vstore_create(int32_t device, int64_t max_actions, int64_t arena_bytes, int32_t max_batch,
                               int64_t max_batch_bytes, ams_vstore_t* out);

/* Interns n actions given as CSR bytes (data host or device; offsets HOST [n+1]).
 * ids_in: DEVICE [n] precomputed ids, or NULL to hash the bytes here (two-phase hash).
 * out_ids (DEVICE u64 [n]) receives the ids, out_status (DEVICE u8 [n]) the status. */
ams_status_t ams_vstore_intern(ams_vstore_t store, const uint8_t* data, const int64_t* offsets, int32_t n,
                               const uint64_t* ids_in, uint64_t* out_ids, uint8_t* out_status, void* stream);

/* Decrements the reference count of n ids (DEVICE [n]); out_remaining (DEVICE i64 [n])
 * gets the remaining count, or -1 for an unknown id (SPEC UnknownId).  At zero the
 * entry is removed. */
ams_status_t ams_vstore_release(ams_vstore_t store, const uint64_t* ids, int32_t n, int64_t* out_remaining,
                                void* stream);

/* Looks up n ids (DEVICE): arena offset and length (DEVICE i64 [n]; -1 if unknown) and,
 * if out_refcount is not NULL, the reference count (0 if unknown).  Offsets stay valid
 * until the next ams_vstore_intern or ams_vstore_compact (either may move bytes). */
ams_status_t ams_vstore_resolve(ams_vstore_t store, const uint64_t* ids, int32_t n, int64_t* out_offset,
                                int64_t* out_len, int64_t* out_refcount, void* stream);

/* Device pointer of the byte arena (read-only for callers). */
ams_status_t ams_vstore_arena(ams_vstore_t store, const uint8_t** arena);

/* Synchronises; live entries, their total bytes, and the arena top (bytes in use,
 * including holes left by removed entries that no compaction has reclaimed yet). */
ams_status_t ams_vstore_stats(ams_vstore_t store, int64_t* n_entries, int64_t* total_bytes, int64_t* arena_used);

/* Reclaims the space of removed entries ("Any action whose reference count
 * drops to zero is removed"; SPEC.md "no leak"): packs the live entries' bytes to the
 * front of the arena (arena top = total live bytes afterwards) and rebuilds the table
 * without tombstones.  ams_vstore_intern runs it automatically when a batch might not fit
 * behind the arena top or might push the table past 3/4 load.  Stream-ordered on
 * `stream`, then synchronises it once.  Resolved offsets become stale.
 * Errors: AMS_ERR_INVALID_ARGUMENT, AMS_ERR_CUDA. */
ams_status_t ams_vstore_compact(ams_vstore_t store, void* stream);

ams_status_t ams_vstore_destroy(ams_vstore_t store);

/* ---- layered storage of action-context blobs ----
 * PAPER.md:497-522 (3.2.2): "we store [frequently accessed data] in GPU memory ... for
 * data that is infrequently accessed, we apply an on-demand recomputation strategy or move
 * it to CPU"; PAPER.md:586-594 (3.2.3 Auto Eviction): LRU combined with priority, "first
 * evict the KV Cache of vision models" (recomputable).  Policy as SPEC.md:200-224
 * (evict_until): victims by ascending P = 1000*class_rank + recency_rank (VisionKV 0 <
 * LlmKV 1 < DiffusionLatent = OutputEmbedding 2; recency rank 0 = least recently used),
 * ties by LRU then id; VisionKV dropped, others demoted to pinned host memory.  Fast tier
 * = HBM (stream-ordered allocations), slow tier = pinned host; copies on `stream`. */
typedef struct ams_tier_s* ams_tier_t;
#define AMS_BLOB_VISION_KV 0
#define AMS_BLOB_LLM_KV 1
#define AMS_BLOB_DIFFUSION_LATENT 2
#define AMS_BLOB_OUTPUT_EMBEDDING 3
#define AMS_TIER_FAST 0
#define AMS_TIER_SLOW 1
#define AMS_TIER_DROPPED 2
#define AMS_EVICT_DEMOTE 1
#define AMS_EVICT_DROP 2
#define AMS_EVICT_PROMOTE 3

/* fast_budget / slow_budget in bytes (slow_budget 0 = unbounded). */
ams_status_t ams_tier_create(int32_t device, int64_t fast_budget, int64_t slow_budget, ams_tier_t* out);

/* Admits a blob (payload host or device, copied on `stream`); placed in HBM when it fits the
 * fast budget (evicting first), otherwise in host memory.  The eviction actions taken are
 * written to act_ids/act_kinds (up to max_acts; *n_acts = total).  Re-admitting a DROPPED
 * blob (after the caller recomputed it) is allowed.  Errors: AMS_ERR_INVALID_ARGUMENT
 * (duplicate live id, bad kind/size), AMS_ERR_CAPACITY (fits no tier; nothing changed),
 * AMS_ERR_OUT_OF_MEMORY, AMS_ERR_CUDA. */
ams_status_t ams_tier_admit(ams_tier_t tier, int64_t blob_id, int32_t kind, const void* payload, int64_t size,
                            int32_t* placed_tier, int64_t* act_ids, int32_t* act_kinds, int32_t max_acts,
                            int32_t* n_acts, void* stream);

/* access_count += 1, last_access = clock++ (SPEC.md:193 touch). */
ams_status_t ams_tier_touch(ams_tier_t tier, int64_t blob_id);

/* Frees >= needed bytes of HBM by the policy above (AMS_ERR_CAPACITY if impossible). */
ams_status_t ams_tier_evict_until(ams_tier_t tier, int64_t needed, int64_t* act_ids, int32_t* act_kinds,
                                  int32_t max_acts, int32_t* n_acts, void* stream);

/* Access: counts as a touch; a host-tier blob is promoted to HBM (evicting as needed);
 * *prev_tier = the tier before the call (AMS_TIER_DROPPED: the caller must recompute and
 * re-admit); *device_ptr = the HBM payload (NULL if not in HBM afterwards). */
ams_status_t ams_tier_fetch(ams_tier_t tier, int64_t blob_id, int32_t* prev_tier, const void** device_ptr,
                            int64_t* act_ids, int32_t* act_kinds, int32_t max_acts, int32_t* n_acts,
                            void* stream);

ams_status_t ams_tier_info(ams_tier_t tier, int64_t blob_id, int32_t* tier_out, int64_t* access_count,
                           int64_t* last_access, int64_t* size);
ams_status_t ams_tier_usage(ams_tier_t tier, int64_t* fast_used, int64_t* slow_used);
/* Copies the current payload (HBM or host tier) to dst (host or device) on `stream`. */
ams_status_t ams_tier_read(ams_tier_t tier, int64_t blob_id, void* dst, void* stream);
ams_status_t ams_tier_destroy(ams_tier_t tier);

/* Number of rows appended so far (global).  Host-side counter, no sync. */
ams_status_t ams_pool_size(ams_pool_t pool, int64_t* n);

/* Synchronises the device, destroys the NCCL communicator (collective if world > 1)
 * and frees everything.  NULL is a no-op. */
ams_status_t ams_pool_destroy(ams_pool_t pool);

/* Static string for a status code. */
const char* ams_status_string(ams_status_t st);

/* ---- instrumentation (bench / tests; not part of the matching semantics) ---- */

/* enable != 0: ams_match records CUDA events (on the caller's stream) around its
 * dominant kernel (the tcgen05 match kernel for bf16, the exact SIMT kernel for fp32). */
ams_status_t ams_pool_set_profiling(ams_pool_t pool, int32_t enable);

/* Waits for the recorded events and returns the summed duration (ms) and number of
 * dominant-kernel launches since the last read, then clears them. */
ams_status_t ams_pool_read_profile(ams_pool_t pool, double* kernel_ms, int64_t* kernel_launches);

/* Total number of CUDA kernels this pool has launched (all entry points). */
ams_status_t ams_pool_launch_count(ams_pool_t pool, int64_t* launches);

/* Describes the last ams_match launch plan: number of row splits, partial lists per
 * query, grid size, dominant-kernel id (0 = fp32 SIMT; 1 = tcgen05, one CTA per
 * 128-query tile; 2 = tcgen05 CTA pair per 256-query tile; 3 = gate-first variant;
 * 4 = tcgen05 small-batch kernel with pool rows on the MMA M side and the nq <= 128
 * queries on N; 5 = as 2, with two CTA pairs per 4-CTA cluster sharing multicast pool
 * rows). Any pointer may be NULL. */
/* Kernel choice for bf16 ams_match calls, for A/B measurements and tests (results are
 * the same either way, within the bf16 tolerances: the small-batch kernel's fp32
 * tensor-core sums of a pair may round differently; the cluster modes are bit-identical).
 * policy is a bit mask, 0 = default:
 *   bit 0 set: batches of nq <= 128 use the 128-query-tile kernel (plan id 1) instead of
 *     the small-batch kernel (plan id 4; used when k <= 32 and round_up(nq, 32) * KT <=
 *     2048, KT = k rounded up to 8/16/32: the per-lane register lists);
 *   bit 1 set: batches with an even number of 256-query tiles use two CTA pairs per
 *     4-CTA cluster sharing multicast pool rows (plan id 5) instead of one pair per
 *     cluster (plan id 2).  Opt-in: only the co-resident 4-CTA clusters are launched
 *     (33 = 132 SMs on a B200), which costs more than the multicast saves;
 *   bit 2 set: the small-batch kernel on CTA pairs (129-256 queries, k <= 8) stages two
 *     256-row tiles per pipeline stage ("wide": every staged query byte serves twice the
 *     pool rows, single-buffered accumulators) instead of one ("narrow", the default:
 *     measured faster);
 *   bit 3 set: ungated batches of 129-256 queries (k <= 8) also use the small-batch CTA
 *     pairs (by default they take the 256-query-tile kernel, measured faster ungated).
 * Host-only; takes effect at the next ams_match.  AMS_ERR_INVALID_ARGUMENT for a NULL
 * pool or a policy outside [0, 15]. */
ams_status_t ams_pool_set_kernel_policy(ams_pool_t pool, int32_t policy);

/* Plan of the last ams_match / ams_match_gate_first / ams_match_auto on this pool (for
 * tests and benchmarks): row splits, partial lists per query, grid size and the kernel:
 * 0 fp32 exact thread-per-row (gated fp32 calls), 1 tcgen05 128-query tiles on one CTA,
 * 2 tcgen05 CTA pairs (256-query tiles), 3 gate-first, 4 small-batch (pool rows on the
 * MMA M side; one CTA or a CTA pair), 5 CTA pairs in 4-CTA multicast clusters, 6 fp32
 * exact tiled (ungated fp32 calls), -1 none yet.  Any output pointer may be NULL. */
ams_status_t ams_pool_last_plan(ams_pool_t pool, int32_t* splits, int32_t* partials,
                                int32_t* grid, int32_t* kernel_id);

/* Shard map (host-only, no device work): owner rank and local row of a global ordinal,
 * for a pool of `capacity` rows over `world` ranks with block size `shard_block`
 * (0 = contiguous).  Returns AMS_ERR_INVALID_ARGUMENT on bad arguments. */
ams_status_t ams_shard_locate(int64_t capacity, int32_t world, int64_t shard_block,
                              int64_t global_index, int32_t* owner, int64_t* local_row);

/* Rows of the global range [0, capacity) owned by `rank` (its shard capacity). */
ams_status_t ams_shard_capacity(int64_t capacity, int32_t world, int64_t shard_block,
                                int32_t rank, int64_t* rows);

int32_t ams_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* AMS_H_ */
