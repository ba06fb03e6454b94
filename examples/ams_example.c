/*
 * ams_example.c -- the C ABI (include/ams.h) used from plain C, no Python: create a pool,
 * record contexts ("adds the unseen vector ... into the context pool"), look
 * them up before an "inference", print the replay decision, destroy.
 *
 *   gcc -O2 -std=c11 examples/ams_example.c -I include -I /usr/local/cuda/include \
 *       -L paper_2508_10259_b200 -l:libams.so -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2508_10259_b200 -o build/ams_example && build/ams_example
 *
 * Pool: 4096 contexts of a 512-wide fp32 embedding + 7 joints (host buffers: the library
 * stages them).  Queries: 8 perturbed copies of stored contexts (hits) + 8 random ones
 * (misses).  Outputs of ams_match are device buffers, copied back with cudaMemcpy.
 * Exit status 0 iff every perturbed query's top-1 is its source row and is a hit, and
 * every random query misses.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "ams.h"

#define CHECK(x)                                                                          \
  do {                                                                                    \
    ams_status_t st_ = (x);                                                               \
    if (st_ != AMS_OK) {                                                                  \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, ams_status_string(st_)); \
      return 1;                                                                           \
    }                                                                                     \
  } while (0)

static uint64_t rng = 88172645463325252ull;
static double uniform(void) {   /* xorshift64*, [0, 1) */
  rng ^= rng >> 12;
  rng ^= rng << 25;
  rng ^= rng >> 27;
  return (double)((rng * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0);
}
static float gauss(void) { return (float)(sqrt(-2.0 * log(uniform() + 1e-300)) * cos(6.283185307179586 * uniform())); }

static void unit(float* v, int d) {
  double s = 0.0;
  for (int t = 0; t < d; ++t) s += (double)v[t] * v[t];
  const float inv = (float)(1.0 / sqrt(s));
  for (int t = 0; t < d; ++t) v[t] *= inv;
}

int main(void) {
  enum { M = 4096, D = 512, J = 7, NQ = 16, K = 4 };
  const float theta = 0.9f, gamma = 0.3f;
  float* emb = (float*)malloc(sizeof(float) * M * D);
  float* joints = (float*)malloc(sizeof(float) * M * J);
  float* q = (float*)malloc(sizeof(float) * NQ * D);
  float* qj = (float*)malloc(sizeof(float) * NQ * J);
  int src[NQ];
  for (int i = 0; i < M; ++i) {
    for (int t = 0; t < D; ++t) emb[(size_t)i * D + t] = gauss();
    unit(emb + (size_t)i * D, D);
    for (int t = 0; t < J; ++t) joints[i * J + t] = (float)(6.283185307179586 * uniform() - 3.141592653589793);
  }
  for (int i = 0; i < NQ; ++i) {
    src[i] = i < NQ / 2 ? (int)(uniform() * M) : -1;
    for (int t = 0; t < D; ++t)
      q[i * D + t] = src[i] >= 0 ? emb[(size_t)src[i] * D + t] + 0.05f / sqrtf((float)D) * gauss() : gauss();
    unit(q + i * D, D);
    for (int t = 0; t < J; ++t)
      qj[i * J + t] = src[i] >= 0 ? joints[src[i] * J + t] + 0.02f * gauss()
                                  : (float)(6.283185307179586 * uniform() - 3.141592653589793);
  }

  ams_pool_config_t cfg = {0};
  cfg.dim = D;
  cfg.joint_dim = J;
  cfg.dtype = AMS_DTYPE_FP32;   /* the bit-exact canonical path */
  cfg.capacity = M;
  cfg.max_queries = NQ;
  cfg.max_k = K;
  cfg.device = 0;
  cfg.rank = 0;
  cfg.world = 1;
  ams_pool_t pool = NULL;
  CHECK(ams_pool_create(&cfg, &pool));
  int64_t first = -1;
  CHECK(ams_pool_append(pool, emb, joints, M, &first, NULL));

  int64_t* d_idx = NULL;
  float* d_score = NULL;
  uint8_t* d_hit = NULL;
  if (cudaMalloc((void**)&d_idx, sizeof(int64_t) * NQ * K) != cudaSuccess ||
      cudaMalloc((void**)&d_score, sizeof(float) * NQ * K) != cudaSuccess ||
      cudaMalloc((void**)&d_hit, NQ) != cudaSuccess)
    return 1;
  CHECK(ams_match(pool, q, qj, NQ, K, theta, gamma, d_idx, d_score, d_hit, NULL));
  int64_t idx[NQ * K];
  float score[NQ * K];
  uint8_t hit[NQ];
  if (cudaMemcpy(idx, d_idx, sizeof idx, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(score, d_score, sizeof score, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(hit, d_hit, sizeof hit, cudaMemcpyDeviceToHost) != cudaSuccess)
    return 1;

  int bad = 0;
  for (int i = 0; i < NQ; ++i) {
    const int ok = src[i] >= 0 ? (hit[i] == 1 && idx[i * K] == src[i]) : (hit[i] == 0);
    bad += !ok;
    printf("query %2d  %-7s  top-1 %6lld  score %+.6f  -> %s\n", i, src[i] >= 0 ? "near" : "random",
           (long long)idx[i * K], (double)score[i * K], hit[i] ? "replay (hit)" : "infer (miss)");
  }
  int64_t n = 0;
  CHECK(ams_pool_size(pool, &n));
  CHECK(ams_pool_destroy(pool));
  cudaFree(d_idx);
  cudaFree(d_score);
  cudaFree(d_hit);
  free(emb);
  free(joints);
  free(q);
  free(qj);
  printf("pool size %lld, build %s: %s\n", (long long)n, ams_build_id(), bad ? "FAILED" : "ok");
  return bad ? 1 : 0;
}
