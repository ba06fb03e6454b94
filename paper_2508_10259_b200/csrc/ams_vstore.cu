// ams_vstore.cu -- virtual-action store on the GPU (second half).
//
// PAPER.md:577-584 (3.2.3): "a virtual action mechanism ... treating the context as a
// series of uniquely numbered actions with independent reference counts.  These actions
// are stored in a contiguous area.  Each context only keeps track of the actions it
// needs by referencing their IDs.  When a new context adds an action, that action's
// reference count increases.  When a context is evicted or deleted, its referenced
// actions each have their reference count decreased.  Any action whose reference count
// drops to zero is removed."  SPEC.md:112-143 (intern / release / resolve): the id is
// the two-phase hash H_final; intern of identical bytes increments the refcount and
// stores the bytes once; intern of different bytes under an existing id is a collision
// (never overwritten); release at zero removes the entry; unknown ids are errors.
//
// Layout: open-addressing table (power-of-two capacity, linear probing) of
// {key = id | 2^63 (0 = empty, 1 = tombstone), refcount, arena offset, length}; bytes in
// one contiguous device arena, allocated by bumping a top pointer.  Removed entries leave
// holes (and tombstones); `compact` reclaims both ("any action whose reference count drops
// to zero is removed"): the live entries' bytes are packed to the front of
// the arena in table-slot order (exclusive scan of the live lengths) through a scratch
// buffer, and the live keys are re-inserted into a fresh table (no tombstones).  It runs
// automatically before an intern whose bytes might not fit behind the top (host-side upper
// bound of the top) or that might push the table past 3/4 load, and on request
// (ams_vstore_compact).  Batched operations, one thread (or warp for byte copies /
// compares) per action, ordered by kernel boundaries on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <new>

#include "../../include/ams.h"

namespace ams {
namespace vs {

constexpr uint64_t kEmpty = 0, kTomb = 1, kTag = uint64_t(1) << 63;

struct Table {
  unsigned long long* key;
  int* ref;
  long long* off;
  long long* len;
  uint64_t mask;
};

__device__ __forceinline__ uint64_t mix(uint64_t h) {   // spread the 61-bit ids over the slots
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  return h;
}

// insert or find; returns slot (or -1 if the table is full); *created = this thread made it
__device__ int64_t find_or_insert(Table t, uint64_t id, bool* created) {
  const unsigned long long key = id | kTag;
  uint64_t s = mix(id) & t.mask;
  for (uint64_t probe = 0; probe <= t.mask; ++probe, s = (s + 1) & t.mask) {
    unsigned long long k = t.key[s];
    if (k == kEmpty) {
      k = atomicCAS(&t.key[s], kEmpty, key);
      if (k == kEmpty) {
        *created = true;
        return (int64_t)s;
      }
    }
    if (k == key) {
      *created = false;
      return (int64_t)s;
    }
  }
  return -1;
}

__device__ int64_t find(Table t, uint64_t id) {
  const unsigned long long key = id | kTag;
  uint64_t s = mix(id) & t.mask;
  for (uint64_t probe = 0; probe <= t.mask; ++probe, s = (s + 1) & t.mask) {
    const unsigned long long k = t.key[s];
    if (k == key) return (int64_t)s;
    if (k == kEmpty) return -1;
  }
  return -1;
}

// status codes (per action)
enum : uint8_t { kNew = 0, kDedup = 1, kCollision = 2, kFull = 3 };

__global__ void intern_keys_kernel(Table t, const uint64_t* __restrict__ ids, int32_t n, int64_t* __restrict__ slot_of,
                                   uint8_t* __restrict__ status) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool created = false;
  const int64_t s = find_or_insert(t, ids[i], &created);
  slot_of[i] = s;
  if (s < 0) {
    status[i] = kFull;
    return;
  }
  if (created) {
    t.off[s] = -1;   // bytes not yet placed (set by the creator in the next kernel)
    t.len[s] = -1;
  }
  atomicAdd(&t.ref[s], 1);
  status[i] = created ? kNew : kDedup;
}

// creators: allocate arena space and copy their bytes (warp per action)
__global__ void intern_copy_kernel(Table t, const uint8_t* __restrict__ data, const int64_t* __restrict__ offsets,
                                   int32_t n, const int64_t* __restrict__ slot_of, uint8_t* __restrict__ status,
                                   uint8_t* __restrict__ arena, unsigned long long* __restrict__ arena_top,
                                   int64_t arena_cap) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n || status[i] != kNew) return;
  const int64_t s = slot_of[i];
  const int64_t len = offsets[i + 1] - offsets[i];
  unsigned long long off = 0;
  if (lane == 0) off = atomicAdd(arena_top, (unsigned long long)len);
  off = __shfl_sync(0xffffffffu, off, 0);
  if ((int64_t)off + len > arena_cap) {   // arena exhausted: the action is not stored
    if (lane == 0) {
      status[i] = kFull;
      t.len[s] = -2;
      if (atomicSub(&t.ref[s], 1) == 1) atomicExch(&t.key[s], kTomb);
    }
    return;
  }
  const uint8_t* src = data + offsets[i];
  for (int64_t b = lane; b < len; b += 32) arena[off + b] = src[b];
  if (lane == 0) {
    t.off[s] = (long long)off;
    t.len[s] = len;
  }
}

// dedup hits: verify identical bytes; a mismatch is a collision (undo the reference)
__global__ void intern_verify_kernel(Table t, const uint8_t* __restrict__ data, const int64_t* __restrict__ offsets,
                                     int32_t n, const int64_t* __restrict__ slot_of, uint8_t* __restrict__ status,
                                     const uint8_t* __restrict__ arena) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n || status[i] != kDedup) return;
  const int64_t s = slot_of[i];
  const int64_t len = offsets[i + 1] - offsets[i];
  if (t.len[s] == -2) {   // its creator in this batch found the arena full
    if (lane == 0) {
      status[i] = kFull;
      if (atomicSub(&t.ref[s], 1) == 1) atomicExch(&t.key[s], kTomb);
    }
    return;
  }
  bool same = t.len[s] == len;
  if (same) {
    const uint8_t* src = data + offsets[i];
    const uint8_t* dst = arena + t.off[s];
    bool diff = false;
    for (int64_t b = lane; b < len; b += 32) diff |= src[b] != dst[b];
    same = !__any_sync(0xffffffffu, diff);
  }
  if (!same && lane == 0) {
    status[i] = kCollision;
    atomicSub(&t.ref[s], 1);
  }
}

__global__ void release_kernel(Table t, const uint64_t* __restrict__ ids, int32_t n, int64_t* __restrict__ remaining) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = find(t, ids[i]);
  if (s < 0) {
    remaining[i] = -1;
    return;
  }
  const int r = atomicSub(&t.ref[s], 1) - 1;
  if (r < 0) {   // over-release within the batch: undo and report as unknown
    atomicAdd(&t.ref[s], 1);
    remaining[i] = -1;
    return;
  }
  if (r == 0) atomicExch(&t.key[s], kTomb);   // removed
  remaining[i] = r;
}

__global__ void resolve_kernel(Table t, const uint64_t* __restrict__ ids, int32_t n, int64_t* __restrict__ out_off,
                               int64_t* __restrict__ out_len, int64_t* __restrict__ out_ref) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = find(t, ids[i]);
  out_off[i] = s < 0 ? -1 : t.off[s];
  out_len[i] = s < 0 ? -1 : t.len[s];
  if (out_ref) out_ref[i] = s < 0 ? 0 : t.ref[s];
}

// ---- compaction ----------------------------------------------------------------------
__device__ __forceinline__ bool live_slot(const Table& t, uint64_t s) {
  return t.key[s] >= kTag && t.ref[s] > 0 && t.len[s] >= 0;
}

constexpr int kScanBlock = 1024;

// per-slot live length -> ex[s]; per-block sums -> bsum[block]
__global__ void __launch_bounds__(kScanBlock) compact_scan_kernel(Table t, long long* __restrict__ ex,
                                                                   long long* __restrict__ bsum) {
  __shared__ long long sh[kScanBlock];
  const uint64_t s = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const long long v = (s <= t.mask && live_slot(t, s)) ? t.len[s] : 0;
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < kScanBlock; o <<= 1) {   // Hillis-Steele inclusive scan
    const long long a = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] += a;
    __syncthreads();
  }
  if (s <= t.mask) ex[s] = sh[threadIdx.x] - v;
  if (threadIdx.x == kScanBlock - 1) bsum[blockIdx.x] = sh[threadIdx.x];
}

// one block: exclusive scan of the block sums in place; bsum[nb] = total live bytes
__global__ void __launch_bounds__(kScanBlock) compact_bsum_kernel(long long* __restrict__ bsum, int nb) {
  __shared__ long long carry;
  __shared__ long long sh[kScanBlock];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += kScanBlock) {
    const int i = base + threadIdx.x;
    const long long v = i < nb ? bsum[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < kScanBlock; o <<= 1) {
      const long long a = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += a;
      __syncthreads();
    }
    if (i < nb) bsum[i] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == kScanBlock - 1) carry += sh[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) bsum[nb] = carry;
}

// warp per slot: live bytes -> scratch at their packed offset; the entry is re-inserted
// into the fresh table `nt` with its new offset
__global__ void compact_move_kernel(Table t, Table nt, const long long* __restrict__ ex,
                                    const long long* __restrict__ bsum, const uint8_t* __restrict__ arena,
                                    uint8_t* __restrict__ scratch, unsigned long long* __restrict__ n_live) {
  const int lane = threadIdx.x & 31;
  const uint64_t s = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s > t.mask || !live_slot(t, s)) return;
  const long long off = ex[s] + bsum[s / kScanBlock];
  const long long len = t.len[s];
  const uint8_t* src = arena + t.off[s];
  for (long long b = lane; b < len; b += 32) scratch[off + b] = src[b];
  if (lane == 0) {
    bool created = false;
    const uint64_t id = (uint64_t)t.key[s] & ~kTag;
    const int64_t ns = find_or_insert(nt, id, &created);   // fresh table, no tombstones: one slot per live key
    if (ns < 0) return;
    nt.ref[ns] = t.ref[s];
    nt.off[ns] = off;
    nt.len[ns] = len;
    atomicAdd(n_live, 1ull);
  }
}

// scratch -> arena (bytes [0, total)); the new top
__global__ void compact_copy_back_kernel(const uint8_t* __restrict__ scratch, uint8_t* __restrict__ arena,
                                         const long long* __restrict__ total_p, unsigned long long* __restrict__ top) {
  const long long total = *total_p;
  const long long n16 = total / 16;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid; i < (uint64_t)n16; i += stride)
    reinterpret_cast<uint4*>(arena)[i] = reinterpret_cast<const uint4*>(scratch)[i];
  for (uint64_t i = (uint64_t)n16 * 16 + tid; i < (uint64_t)total; i += stride) arena[i] = scratch[i];
  if (tid == 0) *top = (unsigned long long)total;
}

__global__ void stats_kernel(Table t, unsigned long long* __restrict__ out) {   // out[0] entries, out[1] bytes
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s <= t.mask; s += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = t.key[s];
    if (k >= kTag && t.ref[s] > 0) {
      atomicAdd(&out[0], 1ull);
      if (t.len[s] > 0) atomicAdd(&out[1], (unsigned long long)t.len[s]);
    }
  }
}

}  // namespace vs
}  // namespace ams

struct ams_vstore_s {
  int32_t device = 0;
  int64_t cap_batch = 0, cap_bytes_batch = 0, arena_cap = 0;
  ams::vs::Table t{};
  ams::vs::Table t2{};            // spare table: compaction re-inserts the live keys here, then swaps
  long long* scan_ex = nullptr;   // [table capacity] packed offsets (compaction)
  long long* scan_bs = nullptr;   // [table capacity / 1024 + 1] block sums, then the total
  // host-side upper bounds since the last compaction (no synchronisation on the fast path):
  int64_t top_bound = 0;          // arena top <= this (every interned byte counted)
  int64_t slots_bound = 0;        // occupied table slots (live + tombstones) <= this
  int64_t compactions = 0;
  uint8_t* arena = nullptr;
  unsigned long long* arena_top = nullptr;
  unsigned long long* stats = nullptr;
  uint64_t* ids = nullptr;        // [cap_batch] computed ids
  int64_t* slot_of = nullptr;     // [cap_batch]
  int64_t* d_offsets = nullptr;   // [cap_batch + 1]
  uint8_t* stage = nullptr;       // [cap_bytes_batch] host-data staging
  int64_t* h_pinned = nullptr;    // [cap_batch + 1]
  cudaEvent_t done = nullptr;
  bool pending = false;
  ams_hasher_t hasher = nullptr;
  bool broken = false;
};

namespace {
void vstore_free(ams_vstore_s* s) {
  if (!s) return;
  void* ptrs[] = {s->t.key, s->t.ref, s->t.off, s->t.len, s->t2.key, s->t2.ref, s->t2.off, s->t2.len, s->scan_ex,
                  s->scan_bs, s->arena, s->arena_top, s->stats, s->ids, s->slot_of, s->d_offsets, s->stage};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (s->h_pinned) cudaFreeHost(s->h_pinned);
  if (s->done) cudaEventDestroy(s->done);
  if (s->hasher) ams_hasher_destroy(s->hasher);
  delete s;
}
// Stream-ordered compaction (see the header comment); synchronises once at the end to
// re-seed the host-side bounds with the exact top and live count.
ams_status_t compact(ams_vstore_s* s, cudaStream_t st) {
  using namespace ams::vs;
  const uint64_t cap = s->t.mask + 1;
  const int nb = (int)((cap + kScanBlock - 1) / kScanBlock);
  uint8_t* scratch = nullptr;
  bool ok = cudaMallocAsync((void**)&scratch, (size_t)std::max<int64_t>(s->arena_cap, 16), st) == cudaSuccess &&
            cudaMemsetAsync(s->t2.key, 0, cap * 8, st) == cudaSuccess &&
            cudaMemsetAsync(s->t2.ref, 0, cap * 4, st) == cudaSuccess &&
            cudaMemsetAsync(s->stats, 0, 16, st) == cudaSuccess;
  if (ok) {
    compact_scan_kernel<<<nb, kScanBlock, 0, st>>>(s->t, s->scan_ex, s->scan_bs);
    compact_bsum_kernel<<<1, kScanBlock, 0, st>>>(s->scan_bs, nb);
    compact_move_kernel<<<(unsigned)((cap + 7) / 8), 256, 0, st>>>(s->t, s->t2, s->scan_ex, s->scan_bs, s->arena,
                                                                  scratch, s->stats);
    compact_copy_back_kernel<<<148 * 4, 256, 0, st>>>(scratch, s->arena, s->scan_bs + nb, s->arena_top);
    ok = cudaGetLastError() == cudaSuccess && cudaFreeAsync(scratch, st) == cudaSuccess;
  }
  unsigned long long top = 0, live = 0;
  ok = ok && cudaMemcpyAsync(&top, s->arena_top, 8, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
       cudaMemcpyAsync(&live, s->stats, 8, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
       cudaStreamSynchronize(st) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    s->broken = true;
    return AMS_ERR_CUDA;
  }
  std::swap(s->t, s->t2);
  s->top_bound = (int64_t)top;
  s->slots_bound = (int64_t)live;
  ++s->compactions;
  return AMS_OK;
}

bool is_dev(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
}  // namespace

extern "C" {

ams_status_t ams_vstore_create(int32_t device, int64_t max_actions, int64_t arena_bytes, int32_t max_batch,
                               int64_t max_batch_bytes, ams_vstore_t* out) {
  if (out == nullptr || max_actions < 1 || arena_bytes < 0 || max_batch < 1 || max_batch_bytes < 0)
    return AMS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return AMS_ERR_INVALID_ARGUMENT;
  }
  if (cudaSetDevice(device) != cudaSuccess) return AMS_ERR_CUDA;
  auto* s = new (std::nothrow) ams_vstore_s;
  if (!s) return AMS_ERR_OUT_OF_MEMORY;
  s->device = device;
  s->cap_batch = max_batch;
  s->cap_bytes_batch = max_batch_bytes;
  s->arena_cap = arena_bytes;
  uint64_t cap = 1024;
  while (cap < (uint64_t)max_actions * 2) cap <<= 1;
  s->t.mask = cap - 1;
  s->t2.mask = cap - 1;
  bool ok = cudaMalloc(&s->t.key, cap * 8) == cudaSuccess && cudaMalloc(&s->t.ref, cap * 4) == cudaSuccess &&
            cudaMalloc(&s->t.off, cap * 8) == cudaSuccess && cudaMalloc(&s->t.len, cap * 8) == cudaSuccess &&
            cudaMalloc(&s->t2.key, cap * 8) == cudaSuccess && cudaMalloc(&s->t2.ref, cap * 4) == cudaSuccess &&
            cudaMalloc(&s->t2.off, cap * 8) == cudaSuccess && cudaMalloc(&s->t2.len, cap * 8) == cudaSuccess &&
            cudaMalloc(&s->scan_ex, cap * 8) == cudaSuccess &&
            cudaMalloc(&s->scan_bs, (cap / 1024 + 2) * 8) == cudaSuccess &&
            cudaMalloc(&s->arena, std::max<int64_t>(arena_bytes, 16)) == cudaSuccess &&
            cudaMalloc(&s->arena_top, 8) == cudaSuccess && cudaMalloc(&s->stats, 16) == cudaSuccess &&
            cudaMalloc(&s->ids, (size_t)max_batch * 8) == cudaSuccess &&
            cudaMalloc(&s->slot_of, (size_t)max_batch * 8) == cudaSuccess &&
            cudaMalloc(&s->d_offsets, ((size_t)max_batch + 1) * 8) == cudaSuccess &&
            cudaMalloc(&s->stage, std::max<int64_t>(max_batch_bytes, 16)) == cudaSuccess &&
            cudaMallocHost(&s->h_pinned, ((size_t)max_batch + 1) * 8) == cudaSuccess &&
            cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaMemset(s->t.key, 0, cap * 8) == cudaSuccess && cudaMemset(s->t.ref, 0, cap * 4) == cudaSuccess &&
       cudaMemset(s->arena_top, 0, 8) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    vstore_free(s);
    return AMS_ERR_OUT_OF_MEMORY;
  }
  const ams_status_t st = ams_hasher_create(device, max_batch, std::max<int64_t>(max_batch_bytes, 1), 4096, &s->hasher);
  if (st != AMS_OK) {
    vstore_free(s);
    return st;
  }
  *out = s;
  return AMS_OK;
}

ams_status_t ams_vstore_intern(ams_vstore_t s, const uint8_t* data, const int64_t* offsets, int32_t n,
                               const uint64_t* ids_in, uint64_t* out_ids, uint8_t* out_status, void* stream) {
  using namespace ams::vs;
  if (s == nullptr || offsets == nullptr || out_ids == nullptr || out_status == nullptr || n < 1 || n > s->cap_batch)
    return AMS_ERR_INVALID_ARGUMENT;
  if (s->broken) return AMS_ERR_CUDA;
  const int64_t total = offsets[n] - offsets[0];
  if (offsets[0] < 0 || total < 0 || (total > 0 && data == nullptr)) return AMS_ERR_INVALID_ARGUMENT;
  if (total > s->cap_bytes_batch) return AMS_ERR_CAPACITY;
  for (int32_t i = 0; i < n; ++i)
    if (offsets[i + 1] < offsets[i]) return AMS_ERR_INVALID_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaSetDevice(s->device) != cudaSuccess) return AMS_ERR_CUDA;
  // ids: caller-supplied (device) or the two-phase hash of each action
  if (ids_in != nullptr) {
    if (cudaMemcpyAsync(out_ids, ids_in, (size_t)n * 8, cudaMemcpyDefault, st) != cudaSuccess) return AMS_ERR_CUDA;
  } else {
    const ams_status_t hs = ams_hash_actions(s->hasher, data, offsets, n, out_ids, stream);
    if (hs != AMS_OK) return hs;
  }
  // reclaim removed entries first if this batch might not fit behind the arena top or
  // might push the table past 3/4 load (host-side upper bounds; exact after compaction)
  const int64_t slot_cap = (int64_t)(s->t.mask + 1);
  if (s->top_bound + total > s->arena_cap || s->slots_bound + n > slot_cap / 4 * 3) {
    const ams_status_t cs = compact(s, st);
    if (cs != AMS_OK) return cs;
  }
  s->top_bound += total;
  s->slots_bound += n;
  // device copies of the bytes (rebased) and offsets
  if (s->pending && cudaEventSynchronize(s->done) != cudaSuccess) return AMS_ERR_CUDA;
  for (int32_t i = 0; i <= n; ++i) s->h_pinned[i] = offsets[i] - offsets[0];
  bool ok = cudaMemcpyAsync(s->d_offsets, s->h_pinned, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, st) == cudaSuccess;
  const uint8_t* src = s->stage;
  if (ok && total > 0) {
    if (is_dev(data))
      src = data + offsets[0];
    else
      ok = cudaMemcpyAsync(s->stage, data + offsets[0], total, cudaMemcpyDefault, st) == cudaSuccess;
  }
  if (ok) {
    intern_keys_kernel<<<(n + 255) / 256, 256, 0, st>>>(s->t, out_ids, n, s->slot_of, out_status);
    intern_copy_kernel<<<(n + 7) / 8, 256, 0, st>>>(s->t, src, s->d_offsets, n, s->slot_of, out_status, s->arena,
                                                    s->arena_top, s->arena_cap);
    intern_verify_kernel<<<(n + 7) / 8, 256, 0, st>>>(s->t, src, s->d_offsets, n, s->slot_of, out_status, s->arena);
    ok = cudaGetLastError() == cudaSuccess && cudaEventRecord(s->done, st) == cudaSuccess;
  }
  if (!ok) {
    s->broken = true;
    return AMS_ERR_CUDA;
  }
  s->pending = true;
  return AMS_OK;
}

ams_status_t ams_vstore_release(ams_vstore_t s, const uint64_t* ids, int32_t n, int64_t* out_remaining, void* stream) {
  if (s == nullptr || ids == nullptr || out_remaining == nullptr || n < 1) return AMS_ERR_INVALID_ARGUMENT;
  if (s->broken) return AMS_ERR_CUDA;
  if (cudaSetDevice(s->device) != cudaSuccess) return AMS_ERR_CUDA;
  ams::vs::release_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(s->t, ids, n, out_remaining);
  if (cudaGetLastError() != cudaSuccess) {
    s->broken = true;
    return AMS_ERR_CUDA;
  }
  return AMS_OK;
}

ams_status_t ams_vstore_resolve(ams_vstore_t s, const uint64_t* ids, int32_t n, int64_t* out_offset, int64_t* out_len,
                                int64_t* out_refcount, void* stream) {
  if (s == nullptr || ids == nullptr || out_offset == nullptr || out_len == nullptr || n < 1)
    return AMS_ERR_INVALID_ARGUMENT;
  if (s->broken) return AMS_ERR_CUDA;
  if (cudaSetDevice(s->device) != cudaSuccess) return AMS_ERR_CUDA;
  ams::vs::resolve_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(s->t, ids, n, out_offset,
                                                                                            out_len, out_refcount);
  if (cudaGetLastError() != cudaSuccess) {
    s->broken = true;
    return AMS_ERR_CUDA;
  }
  return AMS_OK;
}

ams_status_t ams_vstore_compact(ams_vstore_t s, void* stream) {
  if (s == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  if (s->broken) return AMS_ERR_CUDA;
  if (cudaSetDevice(s->device) != cudaSuccess) return AMS_ERR_CUDA;
  return compact(s, static_cast<cudaStream_t>(stream));
}

ams_status_t ams_vstore_arena(ams_vstore_t s, const uint8_t** arena) {
  if (s == nullptr || arena == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  *arena = s->arena;
  return AMS_OK;
}

ams_status_t ams_vstore_stats(ams_vstore_t s, int64_t* n_entries, int64_t* total_bytes, int64_t* arena_used) {
  if (s == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  if (cudaSetDevice(s->device) != cudaSuccess) return AMS_ERR_CUDA;
  unsigned long long h[2] = {0, 0}, top = 0;
  bool ok = cudaDeviceSynchronize() == cudaSuccess && cudaMemset(s->stats, 0, 16) == cudaSuccess;
  if (ok) {
    ams::vs::stats_kernel<<<148 * 4, 256>>>(s->t, s->stats);
    ok = cudaGetLastError() == cudaSuccess && cudaMemcpy(h, s->stats, 16, cudaMemcpyDeviceToHost) == cudaSuccess &&
         cudaMemcpy(&top, s->arena_top, 8, cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  if (!ok) return AMS_ERR_CUDA;
  if (n_entries) *n_entries = (int64_t)h[0];
  if (total_bytes) *total_bytes = (int64_t)h[1];
  if (arena_used) *arena_used = (int64_t)top;
  return AMS_OK;
}

ams_status_t ams_vstore_destroy(ams_vstore_t s) {
  if (s == nullptr) return AMS_OK;
  cudaSetDevice(s->device);
  const ams_status_t st = cudaDeviceSynchronize() == cudaSuccess ? AMS_OK : AMS_ERR_CUDA;
  vstore_free(s);
  return st;
}

}  // extern "C"
