// ams_tier.cu -- layered storage of action-context blobs with auto-eviction
// (PAPER.md:497-522 3.2.2 and PAPER.md:586-594 3.2.3).
//
// Fast tier = HBM (stream-ordered cudaMallocAsync blocks), slow tier = pinned host memory.
// Policy (identical to oracle/tier.py): admit into HBM when the blob fits
// the fast budget, evicting first if needed, else into host memory; victims in ascending
// P = 1000*class_rank + recency_rank (VisionKV 0 < LlmKV 1 < DiffusionLatent =
// OutputEmbedding 2; recency rank 0 = least recently used), ties by LRU then id; VisionKV
// is dropped ("can be easily recalculated"), everything else demoted to
// host memory (device->host copy on the caller's stream); a fetched host blob is promoted
// back (host->device copy), evicting as needed.  Host control logic in C++; the data
// movement is async copies ordered on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <new>
#include <tuple>
#include <vector>

#include "../../include/ams.h"

namespace {

struct Blob {
  int32_t kind = 0;
  int64_t size = 0;
  int32_t tier = AMS_TIER_FAST;
  int64_t count = 0, last = 0;
  void* dev = nullptr;    // HBM copy (tier FAST)
  void* host = nullptr;   // pinned host copy (tier SLOW)
};

struct Pending {         // host buffer to free once `ev` completes
  void* host;
  cudaEvent_t ev;
};

int class_rank(int kind) { return kind == AMS_BLOB_VISION_KV ? 0 : kind == AMS_BLOB_LLM_KV ? 1 : 2; }

}  // namespace

struct ams_tier_s {
  int32_t device = 0;
  int64_t fast_budget = 0, slow_budget = 0, fast_used = 0, slow_used = 0, clock = 0;
  std::map<int64_t, Blob> blobs;
  std::vector<Pending> pending;
  bool broken = false;

  void reap(bool wait) {
    std::vector<Pending> keep;
    for (auto& p : pending) {
      if (wait) cudaEventSynchronize(p.ev);
      if (cudaEventQuery(p.ev) == cudaSuccess) {
        cudaFreeHost(p.host);
        cudaEventDestroy(p.ev);
      } else {
        cudaGetLastError();
        keep.push_back(p);
      }
    }
    pending.swap(keep);
  }

  // victims in eviction order: (P, last, id) ascending over fast-resident blobs
  std::vector<int64_t> victims() const {
    std::vector<std::pair<int64_t, int64_t>> rec;   // (last, id)
    for (auto& kv : blobs)
      if (kv.second.tier == AMS_TIER_FAST) rec.emplace_back(kv.second.last, kv.first);
    std::sort(rec.begin(), rec.end());
    std::vector<std::tuple<int64_t, int64_t, int64_t>> order;   // (P, last, id)
    for (size_t r = 0; r < rec.size(); ++r) {
      const Blob& b = blobs.at(rec[r].second);
      order.emplace_back((int64_t)1000 * class_rank(b.kind) + (int64_t)r, b.last, rec[r].second);
    }
    std::sort(order.begin(), order.end());
    std::vector<int64_t> ids;
    for (auto& o : order) ids.push_back(std::get<2>(o));
    return ids;
  }
};

namespace {

struct Acts {
  int64_t* ids;
  int32_t* kinds;
  int32_t max, n;
  void add(int64_t id, int32_t k) {
    if (ids && kinds && n < max) {
      ids[n] = id;
      kinds[n] = k;
    }
    ++n;
  }
};

// Plans then executes evict_until(needed).  Returns AMS_ERR_CAPACITY with no change.
ams_status_t evict_until(ams_tier_s* t, int64_t needed, Acts& acts, cudaStream_t s) {
  if (needed <= 0) return AMS_OK;
  if (t->fast_used < needed) return AMS_ERR_CAPACITY;
  std::vector<std::pair<int64_t, int32_t>> plan;
  int64_t freed = 0, slow_add = 0;
  for (int64_t id : t->victims()) {
    if (freed >= needed) break;
    const Blob& b = t->blobs.at(id);
    const int32_t a = b.kind == AMS_BLOB_VISION_KV ? AMS_EVICT_DROP : AMS_EVICT_DEMOTE;
    plan.emplace_back(id, a);
    freed += b.size;
    if (a == AMS_EVICT_DEMOTE) slow_add += b.size;
  }
  if (t->slow_budget > 0 && t->slow_used + slow_add > t->slow_budget) return AMS_ERR_CAPACITY;
  for (auto& pa : plan) {
    Blob& b = t->blobs.at(pa.first);
    if (pa.second == AMS_EVICT_DEMOTE) {
      if (cudaMallocHost(&b.host, std::max<int64_t>(b.size, 1)) != cudaSuccess) return AMS_ERR_OUT_OF_MEMORY;
      if (b.size > 0 && cudaMemcpyAsync(b.host, b.dev, b.size, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return AMS_ERR_CUDA;
      b.tier = AMS_TIER_SLOW;
      t->slow_used += b.size;
    } else {
      b.tier = AMS_TIER_DROPPED;
    }
    if (cudaFreeAsync(b.dev, s) != cudaSuccess) return AMS_ERR_CUDA;
    b.dev = nullptr;
    t->fast_used -= b.size;
    acts.add(pa.first, pa.second);
  }
  return AMS_OK;
}

ams_status_t fail(ams_tier_s* t, ams_status_t st) {
  if (st == AMS_ERR_CUDA) t->broken = true;
  return st;
}

}  // namespace

extern "C" {

ams_status_t ams_tier_create(int32_t device, int64_t fast_budget, int64_t slow_budget, ams_tier_t* out) {
  if (out == nullptr || fast_budget < 0 || slow_budget < 0) return AMS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return AMS_ERR_INVALID_ARGUMENT;
  }
  auto* t = new (std::nothrow) ams_tier_s;
  if (!t) return AMS_ERR_OUT_OF_MEMORY;
  t->device = device;
  t->fast_budget = fast_budget;
  t->slow_budget = slow_budget;
  *out = t;
  return AMS_OK;
}

ams_status_t ams_tier_admit(ams_tier_t t, int64_t blob_id, int32_t kind, const void* payload, int64_t size,
                            int32_t* placed_tier, int64_t* act_ids, int32_t* act_kinds, int32_t max_acts,
                            int32_t* n_acts, void* stream) {
  if (t == nullptr || kind < 0 || kind > 3 || size < 0 || (size > 0 && payload == nullptr))
    return AMS_ERR_INVALID_ARGUMENT;
  if (t->broken) return AMS_ERR_CUDA;
  auto it = t->blobs.find(blob_id);
  if (it != t->blobs.end() && it->second.tier != AMS_TIER_DROPPED) return AMS_ERR_INVALID_ARGUMENT;
  if (cudaSetDevice(t->device) != cudaSuccess) return AMS_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  t->reap(false);
  Acts acts{act_ids, act_kinds, max_acts, 0};
  Blob b;
  b.kind = kind;
  b.size = size;
  if (size <= t->fast_budget) {
    const ams_status_t st = evict_until(t, t->fast_used + size - t->fast_budget, acts, s);
    if (st != AMS_OK) return fail(t, st);
    if (cudaMallocAsync(&b.dev, std::max<int64_t>(size, 1), s) != cudaSuccess) return fail(t, AMS_ERR_OUT_OF_MEMORY);
    if (size > 0 && cudaMemcpyAsync(b.dev, payload, size, cudaMemcpyDefault, s) != cudaSuccess)
      return fail(t, AMS_ERR_CUDA);
    b.tier = AMS_TIER_FAST;
    t->fast_used += size;
  } else {
    if (t->slow_budget > 0 && t->slow_used + size > t->slow_budget) return AMS_ERR_CAPACITY;
    if (cudaMallocHost(&b.host, std::max<int64_t>(size, 1)) != cudaSuccess) return AMS_ERR_OUT_OF_MEMORY;
    if (size > 0 && cudaMemcpyAsync(b.host, payload, size, cudaMemcpyDefault, s) != cudaSuccess)
      return fail(t, AMS_ERR_CUDA);
    b.tier = AMS_TIER_SLOW;
    t->slow_used += size;
  }
  b.last = t->clock++;
  t->blobs[blob_id] = b;
  if (placed_tier) *placed_tier = b.tier;
  if (n_acts) *n_acts = acts.n;
  return AMS_OK;
}

ams_status_t ams_tier_touch(ams_tier_t t, int64_t blob_id) {
  if (t == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  auto it = t->blobs.find(blob_id);
  if (it == t->blobs.end()) return AMS_ERR_INVALID_ARGUMENT;
  it->second.count += 1;
  it->second.last = t->clock++;
  return AMS_OK;
}

ams_status_t ams_tier_evict_until(ams_tier_t t, int64_t needed, int64_t* act_ids, int32_t* act_kinds,
                                  int32_t max_acts, int32_t* n_acts, void* stream) {
  if (t == nullptr || needed < 0) return AMS_ERR_INVALID_ARGUMENT;
  if (t->broken) return AMS_ERR_CUDA;
  if (cudaSetDevice(t->device) != cudaSuccess) return AMS_ERR_CUDA;
  Acts acts{act_ids, act_kinds, max_acts, 0};
  const ams_status_t st = evict_until(t, needed, acts, static_cast<cudaStream_t>(stream));
  if (n_acts) *n_acts = acts.n;
  return fail(t, st);
}

ams_status_t ams_tier_fetch(ams_tier_t t, int64_t blob_id, int32_t* prev_tier, const void** device_ptr,
                            int64_t* act_ids, int32_t* act_kinds, int32_t max_acts, int32_t* n_acts, void* stream) {
  if (t == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  if (t->broken) return AMS_ERR_CUDA;
  auto it = t->blobs.find(blob_id);
  if (it == t->blobs.end()) return AMS_ERR_INVALID_ARGUMENT;
  if (cudaSetDevice(t->device) != cudaSuccess) return AMS_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  t->reap(false);
  Acts acts{act_ids, act_kinds, max_acts, 0};
  Blob& b = it->second;
  const int32_t prev = b.tier;
  if (prev_tier) *prev_tier = prev;
  if (prev != AMS_TIER_DROPPED) {
    b.count += 1;
    b.last = t->clock++;
  }
  if (prev == AMS_TIER_SLOW && b.size <= t->fast_budget) {
    const ams_status_t st = evict_until(t, t->fast_used + b.size - t->fast_budget, acts, s);
    if (st != AMS_OK) return fail(t, st);
    if (cudaMallocAsync(&b.dev, std::max<int64_t>(b.size, 1), s) != cudaSuccess) return fail(t, AMS_ERR_OUT_OF_MEMORY);
    if (b.size > 0 && cudaMemcpyAsync(b.dev, b.host, b.size, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return fail(t, AMS_ERR_CUDA);
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(ev, s) != cudaSuccess)
      return fail(t, AMS_ERR_CUDA);
    t->pending.push_back({b.host, ev});   // freed once the copy has run
    b.host = nullptr;
    b.tier = AMS_TIER_FAST;
    t->slow_used -= b.size;
    t->fast_used += b.size;
    acts.add(blob_id, AMS_EVICT_PROMOTE);
  }
  if (device_ptr) *device_ptr = b.tier == AMS_TIER_FAST ? b.dev : nullptr;
  if (n_acts) *n_acts = acts.n;
  return AMS_OK;
}

ams_status_t ams_tier_info(ams_tier_t t, int64_t blob_id, int32_t* tier, int64_t* access_count, int64_t* last_access,
                           int64_t* size) {
  if (t == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  auto it = t->blobs.find(blob_id);
  if (it == t->blobs.end()) return AMS_ERR_INVALID_ARGUMENT;
  if (tier) *tier = it->second.tier;
  if (access_count) *access_count = it->second.count;
  if (last_access) *last_access = it->second.last;
  if (size) *size = it->second.size;
  return AMS_OK;
}

ams_status_t ams_tier_usage(ams_tier_t t, int64_t* fast_used, int64_t* slow_used) {
  if (t == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  if (fast_used) *fast_used = t->fast_used;
  if (slow_used) *slow_used = t->slow_used;
  return AMS_OK;
}

ams_status_t ams_tier_read(ams_tier_t t, int64_t blob_id, void* dst, void* stream) {
  if (t == nullptr || dst == nullptr) return AMS_ERR_INVALID_ARGUMENT;
  auto it = t->blobs.find(blob_id);
  if (it == t->blobs.end() || it->second.tier == AMS_TIER_DROPPED) return AMS_ERR_INVALID_ARGUMENT;
  if (cudaSetDevice(t->device) != cudaSuccess) return AMS_ERR_CUDA;
  const Blob& b = it->second;
  const void* src = b.tier == AMS_TIER_FAST ? b.dev : b.host;
  if (b.size > 0 && cudaMemcpyAsync(dst, src, b.size, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return fail(t, AMS_ERR_CUDA);
  return AMS_OK;
}

ams_status_t ams_tier_destroy(ams_tier_t t) {
  if (t == nullptr) return AMS_OK;
  cudaSetDevice(t->device);
  ams_status_t st = cudaDeviceSynchronize() == cudaSuccess ? AMS_OK : AMS_ERR_CUDA;
  t->reap(true);
  for (auto& kv : t->blobs) {
    if (kv.second.dev) cudaFree(kv.second.dev);
    if (kv.second.host) cudaFreeHost(kv.second.host);
  }
  delete t;
  return st;
}

}  // extern "C"
