// ams_topk.cuh -- per-thread register top-k lists ordered by (score desc, index asc).
//
// North_star: "a warp-shuffle/shared-memory per-query running top-k so the full score
// matrix never reaches HBM"; tie rule "ties go to the lowest index" (reading R4).
// Every array index below is a compile-time constant after unrolling (no local memory).
#pragma once
#include <cstdint>
#include <math_constants.h>

namespace ams {

template <typename I>
__device__ __forceinline__ bool better(float s, I i, float t, I j) {
  // (s, i) ranks strictly before (t, j); padding is (-inf, -1) and ranks last
  return s > t || (s == t && i >= 0 && (j < 0 || i < j));
}

template <int KT, typename I>
struct TopK {
  float s[KT];
  I i[KT];
  float kth_s;   // k-th best score (the admission threshold)
  I kth_i;

  __device__ __forceinline__ void init(bool active) {
#pragma unroll
    for (int r = 0; r < KT; ++r) {
      s[r] = -CUDART_INF_F;
      i[r] = I(-1);
    }
    kth_s = active ? -CUDART_INF_F : CUDART_INF_F;
    kth_i = I(-1);
  }

  // Admission threshold = the last slot (static index: a runtime s[k-1] would be lowered
  // to local memory).  With k < KT this admits more than necessary, never fewer: a
  // candidate that does not beat the KT-th best cannot be in the top k.
  __device__ __forceinline__ void refresh_kth(int /*k*/) {
    kth_s = s[KT - 1];
    kth_i = i[KT - 1];
  }

  // Insert (v, j) whose index is larger than every index held (monotone scan): ties
  // with held scores go after them.  Caller guarantees v > kth_s.
  __device__ __forceinline__ void insert_monotone(float v, I j, int k) {
#pragma unroll
    for (int r = KT - 1; r >= 0; --r) {
      const float ps = r > 0 ? s[r > 0 ? r - 1 : 0] : CUDART_INF_F;
      const I pi = r > 0 ? i[r > 0 ? r - 1 : 0] : I(0);
      const bool gp = v > ps;
      const bool gc = v > s[r];
      s[r] = gp ? ps : (gc ? v : s[r]);
      i[r] = gp ? pi : (gc ? j : i[r]);
    }
    refresh_kth(k);
  }

  // General insert by (score desc, index asc).  Caller guarantees better(v, j, kth).
  __device__ __forceinline__ void insert(float v, I j, int k) {
#pragma unroll
    for (int r = KT - 1; r >= 0; --r) {
      const bool has_prev = r > 0;
      const float ps = has_prev ? s[r > 0 ? r - 1 : 0] : CUDART_INF_F;
      const I pi = has_prev ? i[r > 0 ? r - 1 : 0] : I(-2);
      const bool gp = has_prev && better(v, j, ps, pi);
      const bool gc = better(v, j, s[r], i[r]);
      s[r] = gp ? ps : (gc ? v : s[r]);
      i[r] = gp ? pi : (gc ? j : i[r]);
    }
    refresh_kth(k);
  }

  __device__ __forceinline__ void pop_front() {
#pragma unroll
    for (int r = 0; r < KT - 1; ++r) {
      s[r] = s[r + 1];
      i[r] = i[r + 1];
    }
    s[KT - 1] = -CUDART_INF_F;
    i[KT - 1] = I(-1);
  }
};

}  // namespace ams
