/*
 * ams_oracle.c -- CPU brute-force oracle for AMS action-context matching.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  The
 * product path (paper_2508_10259_b200/) never links, imports or executes it, and
 * this file shares no code, header, table or helper with the CUDA path.
 *
 * What it computes (the plain definition of the matching step; DESIGN.md
 * "Oracle" and SURVEY.md 8(c)):
 *   PAPER.md:486 (3.2.1)  a pool context = output embedding + robot joint state;
 *   PAPER.md:489 (3.2.1)  before inference, "checks the action context pool to see
 *                         if any similar and reusable intermediate states exist";
 *   PAPER.md:865 (4)      stored contexts are retrieved "one by one" -> a ranked list;
 *   SPEC.md:186-190       lookup returns the best match "or none below threshold";
 *   BASELINE.json north_star: cosine similarity over the embedding, gated by the
 *                         L2 joint distance, per-query top-k, threshold -> hit flag,
 *                         ties to the lowest index.
 *
 * For every query i and pool row j (global append ordinal):
 *   1 norms   bf16: exact decode to fp64, n = sqrt(sum x^2) in fp64, inv = n>0 ? 1/n : 0
 *             fp32: ss = fmaf chain in ascending t; inv = ss>0 ? 1.0f/sqrtf(ss) : 0.0f
 *   2 dot     bf16: fp64 sum (ascending t) of exact bf16*bf16 products
 *             fp32: acc = fmaf(q_t, e_t, acc), t ascending
 *   3 score   s = (dot * inv_q) * inv_e, left to right (fp64 for bf16, fp32 for fp32)
 *   4 gate    canonical fp32 for both dtypes: ds = +0; for t: diff = r_t - p_t;
 *             ds = fmaf(diff, diff, ds); eligible iff ds <= g2, g2 = fp32(gamma*gamma)
 *   5 select  eligible rows sorted by (s desc, global id asc); first min(k, n_elig),
 *             pad (-1, -inf)
 *   6 hit     n_elig >= 1 && s_top1 >= theta     ("none below threshold")
 * Readings R1-R21 are listed in DESIGN.md.
 *
 * Mode A: brute force over all pairs.  Mode B: scan the gate for every pair first,
 * then score only eligible pairs -- identical by definition (ineligible rows never
 * enter step 5); it exists so full-Q gated parity is affordable on host cores.
 *
 * Compile: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC
 * (no contraction: every fp32 multiply/add above rounds where the definition says).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_BF16 0
#define ORC_FP32 1

static double bf16_decode(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return (double)f;
}

/* step 1, bf16 */
void oracle_inv_norm_bf16(const uint16_t* x, int64_t n, int32_t d, double* inv) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int32_t t = 0; t < d; ++t) {
      double v = bf16_decode(x[i * d + t]);
      s += v * v;
    }
    double nr = sqrt(s);
    inv[i] = nr > 0.0 ? 1.0 / nr : 0.0;
  }
}

/* step 1, fp32 canonical */
void oracle_inv_norm_f32(const float* x, int64_t n, int32_t d, float* inv) {
  for (int64_t i = 0; i < n; ++i) {
    float ss = 0.0f;
    for (int32_t t = 0; t < d; ++t) ss = fmaf(x[i * d + t], x[i * d + t], ss);
    inv[i] = ss > 0.0f ? 1.0f / sqrtf(ss) : 0.0f;
  }
}

/* step 4: returns ds; eligibility is (ds <= g2) */
float oracle_gate_ds(const float* r, const float* p, int32_t J) {
  float ds = 0.0f;
  for (int32_t t = 0; t < J; ++t) {
    float diff = r[t] - p[t];
    ds = fmaf(diff, diff, ds);
  }
  return ds;
}

float oracle_gate_g2(float gamma) {
  float g2 = gamma * gamma;
  return g2;
}

/* step 2 + 3 */
static double score_bf16(const uint16_t* q, const uint16_t* e, int32_t d, double inv_q, double inv_e) {
  double dot = 0.0;
  for (int32_t t = 0; t < d; ++t) dot += bf16_decode(q[t]) * bf16_decode(e[t]);
  return (dot * inv_q) * inv_e;
}

static float score_f32(const float* q, const float* e, int32_t d, float inv_q, float inv_e) {
  float acc = 0.0f;
  for (int32_t t = 0; t < d; ++t) acc = fmaf(q[t], e[t], acc);
  float s = acc * inv_q;
  s = s * inv_e;
  return s;
}

typedef struct {
  double s;   /* ranking key: fp64 score (bf16) or the fp32 score widened exactly (fp32) */
  int64_t id; /* global append ordinal */
} cand_t;

/* step 5 order: s descending, id ascending */
static int cand_cmp(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->s > y->s) return -1;
  if (x->s < y->s) return 1;
  if (x->id < y->id) return -1;
  if (x->id > y->id) return 1;
  return 0;
}

/*
 * oracle_match: all pool rows vs all queries.
 *   dtype      ORC_BF16 (emb/q_emb are uint16 bf16 bits) or ORC_FP32 (float)
 *   emb        [M, d] row-major; joints [M, J] fp32
 *   row_ids    [M] global ids of the rows, or NULL (row j has id j)
 *   q_emb      [nq, d]; q_joints [nq, J]
 *   mode       0 = A (brute force), 1 = B (gate first)
 *   outputs    out_idx [nq,k] int64, out_score [nq,k] fp32, out_hit [nq] u8,
 *              optional: out_score64 [nq,k] (ranking key), out_next [nq] ((k+1)-th
 *              ranking key or -inf), out_nelig [nq]
 * Returns 0 on success, -1 on bad arguments or allocation failure.
 */
int oracle_match(int32_t dtype, const void* emb, const float* joints, const int64_t* row_ids,
                 int64_t M, int32_t d, int32_t J, const void* q_emb, const float* q_joints,
                 int32_t nq, int32_t k, float theta, float gamma, int32_t mode, int32_t nthreads,
                 int64_t* out_idx, float* out_score, uint8_t* out_hit, double* out_score64,
                 double* out_next, int64_t* out_nelig) {
  if (nq < 0 || k < 1 || M < 0 || d < 1 || J < 1) return -1;
  if (dtype != ORC_BF16 && dtype != ORC_FP32) return -1;
  const float g2 = oracle_gate_g2(gamma);

  double* inv_e64 = NULL;
  double* inv_q64 = NULL;
  float* inv_e32 = NULL;
  float* inv_q32 = NULL;
  if (dtype == ORC_BF16) {
    inv_e64 = (double*)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1));
    inv_q64 = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1));
    if (!inv_e64 || !inv_q64) { free(inv_e64); free(inv_q64); return -1; }
    oracle_inv_norm_bf16((const uint16_t*)emb, M, d, inv_e64);
    oracle_inv_norm_bf16((const uint16_t*)q_emb, nq, d, inv_q64);
  } else {
    inv_e32 = (float*)malloc(sizeof(float) * (size_t)(M > 0 ? M : 1));
    inv_q32 = (float*)malloc(sizeof(float) * (size_t)(nq > 0 ? nq : 1));
    if (!inv_e32 || !inv_q32) { free(inv_e32); free(inv_q32); return -1; }
    oracle_inv_norm_f32((const float*)emb, M, d, inv_e32);
    oracle_inv_norm_f32((const float*)q_emb, nq, d, inv_q32);
  }

  int failed = 0;
#ifdef _OPENMP
  if (nthreads < 1) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
  for (int32_t i = 0; i < nq; ++i) {
    cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)(M > 0 ? M : 1));
    if (!c) { failed = 1; continue; }
    int64_t n = 0;
    const float* r = q_joints + (int64_t)i * J;
    for (int64_t j = 0; j < M; ++j) {
      const float* p = joints + j * J;
      if (mode == 1) { /* B: gate first */
        if (!(oracle_gate_ds(r, p, J) <= g2)) continue;
      }
      double s;
      if (dtype == ORC_BF16)
        s = score_bf16((const uint16_t*)q_emb + (int64_t)i * d, (const uint16_t*)emb + j * d, d,
                       inv_q64[i], inv_e64[j]);
      else
        s = (double)score_f32((const float*)q_emb + (int64_t)i * d, (const float*)emb + j * d, d,
                              inv_q32[i], inv_e32[j]);
      if (mode != 1) { /* A: gate after scoring, same eligibility */
        if (!(oracle_gate_ds(r, p, J) <= g2)) continue;
      }
      c[n].s = s;
      c[n].id = row_ids ? row_ids[j] : j;
      ++n;
    }
    qsort(c, (size_t)n, sizeof(cand_t), cand_cmp);
    for (int32_t r_ = 0; r_ < k; ++r_) {
      int64_t o = (int64_t)i * k + r_;
      if (r_ < n) {
        out_idx[o] = c[r_].id;
        out_score[o] = (float)c[r_].s;
        if (out_score64) out_score64[o] = c[r_].s;
      } else {
        out_idx[o] = -1;
        out_score[o] = -INFINITY;
        if (out_score64) out_score64[o] = -INFINITY;
      }
    }
    if (out_next) out_next[i] = (n > k) ? c[k].s : -INFINITY;
    if (out_nelig) out_nelig[i] = n;
    out_hit[i] = (uint8_t)((n >= 1 && c[0].s >= (double)theta) ? 1 : 0);
    free(c);
  }
  free(inv_e64); free(inv_q64); free(inv_e32); free(inv_q32);
  return failed ? -1 : 0;
}

/*
 * oracle_merge: per query, merge G ranked lists (e.g. per-shard oracle outputs)
 * into the top-k by (key desc, id asc); entries with id < 0 are padding.
 *   keys/ids [G, nq, kin]; outputs [nq, k]; out_hit from the top-1 key vs theta.
 * Plain definition: concatenate, sort, take k (a shard's exact
 * top-k contains every global top-k member that lives in it).
 */
int oracle_merge(const double* keys, const int64_t* ids, int32_t G, int32_t nq, int32_t kin,
                 int32_t k, float theta, int64_t* out_idx, float* out_score, uint8_t* out_hit,
                 double* out_score64) {
  cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)(G * kin > 0 ? G * kin : 1));
  if (!c) return -1;
  for (int32_t i = 0; i < nq; ++i) {
    int64_t n = 0;
    for (int32_t g = 0; g < G; ++g)
      for (int32_t r = 0; r < kin; ++r) {
        int64_t o = ((int64_t)g * nq + i) * kin + r;
        if (ids[o] < 0) continue;
        c[n].s = keys[o];
        c[n].id = ids[o];
        ++n;
      }
    qsort(c, (size_t)n, sizeof(cand_t), cand_cmp);
    for (int32_t r = 0; r < k; ++r) {
      int64_t o = (int64_t)i * k + r;
      out_idx[o] = r < n ? c[r].id : -1;
      out_score[o] = r < n ? (float)c[r].s : -INFINITY;
      if (out_score64) out_score64[o] = r < n ? c[r].s : -INFINITY;
    }
    out_hit[i] = (uint8_t)((n >= 1 && c[0].s >= (double)theta) ? 1 : 0);
  }
  free(c);
  return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------------------
 * Two-phase hashing for the action index (3.2.3, Algorithm 1
 * `lst:impl:index` at PAPER.md:545-574), concretised by SPEC.md:103-111:
 *   Phase 1: partition the N input bytes into k = ceil(N/s) segments of s bytes (the
 *            last may be shorter); h_i = polynomial hash of segment i:
 *            h = 0; for each byte b: h = (h*B + b) mod M.
 *   Phase 2: H_final = fold over i = 1..k of acc = (acc*B + h_i) mod M, from 0.
 * B = 257, M = 2^61 - 1.  Empty input -> 0.
 * Plain sequential definition, one byte at a time, in the paper's order.
 * ------------------------------------------------------------------------------------ */
#define ORC_HASH_M ((((uint64_t)1) << 61) - 1)

static uint64_t mulmod61(uint64_t a, uint64_t b) {
  unsigned __int128 p = (unsigned __int128)a * b;
  return (uint64_t)(p % ORC_HASH_M);
}

uint64_t oracle_hash_segment(const uint8_t* data, int64_t n, uint64_t B) {
  uint64_t h = 0;
  for (int64_t i = 0; i < n; ++i) h = (mulmod61(h, B) + data[i]) % ORC_HASH_M;
  return h;
}

uint64_t oracle_hash_action(const uint8_t* data, int64_t n, int64_t s, uint64_t B) {
  if (n <= 0 || s <= 0) return 0;
  uint64_t acc = 0;
  for (int64_t off = 0; off < n; off += s) {
    int64_t len = (n - off < s) ? (n - off) : s;
    uint64_t h = oracle_hash_segment(data + off, len, B);
    acc = (mulmod61(acc, B) + h) % ORC_HASH_M;
  }
  return acc;
}

/* batch form: inputs [offsets[i], offsets[i+1]) of `data` */
void oracle_hash_actions(const uint8_t* data, const int64_t* offsets, int32_t n_inputs, int64_t s, uint64_t B,
                         uint64_t* out) {
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int32_t i = 0; i < n_inputs; ++i)
    out[i] = oracle_hash_action(data + offsets[i], offsets[i + 1] - offsets[i], s, B);
}
