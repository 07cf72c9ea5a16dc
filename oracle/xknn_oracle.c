/*
 * xknn_oracle.c -- CPU restatement of the reference KNN-softmax hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_2102_06025_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product never links it and
 * never falls back to it.
 *
 * Parity pin: every function below is checked against the reference itself
 * (oracle/_ref/libxcls_ref.so, compiled from /root/reference/proj/src by
 * `make -C oracle ref`, oracle/Makefile) on seeded random inputs and against the SPEC.md
 * known-answer examples and the golden fixtures (tests/test_oracle.py, tests/golden/).
 *
 * Arithmetic is restated operation-for-operation (same loop order, same
 * float/double promotions, no FMA contraction: build with -ffp-contract=off)
 * so that it is bit-identical with the reference built with the same flags.
 *
 * Reference files cited as  <file>:<line>  are relative to /root/reference/proj.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "xknn_oracle.h"

/* ------------------------------------------------------------------------- */
/* mt19937_64 (standard-defined; libstdc++ <random>) and libstdc++ 13's       */
/* uniform_int_distribution<size_t> (Lemire nearly-divisionless, __int128).   */
/* Used by finish_selection's padding draw, knn_softmax.cpp:43-49.            */
/* ------------------------------------------------------------------------- */
#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t mt[MT_N];
  int idx;
  /* test hook: a caller-given word stream replaces the engine's output (or_*_stream) */
  const uint64_t* inj;
  uint64_t inj_len, inj_pos;
} mt64_t;

/* set by or_select_active_shards_stream for the duration of one selection */
static const uint64_t* g_inj_words = NULL;
static uint64_t g_inj_len = 0;

void or_mt64_seed(mt64_t* g, uint64_t seed) {
  g->inj = g_inj_words;
  g->inj_len = g_inj_len;
  g->inj_pos = 0;
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = MT_N;
}

static void mt64_twist(mt64_t* g) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  uint64_t* mt = g->mt;
  int k;
  for (k = 0; k < MT_N - MT_M; ++k) {
    uint64_t y = (mt[k] & UM) | (mt[k + 1] & LM);
    mt[k] = mt[k + MT_M] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
  }
  for (; k < MT_N - 1; ++k) {
    uint64_t y = (mt[k] & UM) | (mt[k + 1] & LM);
    mt[k] = mt[k + (MT_M - MT_N)] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
  }
  uint64_t y = (mt[MT_N - 1] & UM) | (mt[0] & LM);
  mt[MT_N - 1] = mt[MT_M - 1] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
  g->idx = 0;
}

uint64_t or_mt64_next(mt64_t* g) {
  if (g->inj) return g->inj_pos < g->inj_len ? g->inj[g->inj_pos++] : 0;
  if (g->idx >= MT_N) mt64_twist(g);
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= (z >> 43);
  return z;
}

/* uniform_int_distribution<size_t>(a, b)(g): /usr/include/c++/13/bits/uniform_int_dist.h:257-274,305-320 */
uint64_t or_uniform_u64(mt64_t* g, uint64_t a, uint64_t b) {
  const uint64_t range = b - a + 1;  /* __uerange; b - a < 2^64-1 always here */
  unsigned __int128 prod = (unsigned __int128)or_mt64_next(g) * range;
  uint64_t low = (uint64_t)prod;
  if (low < range) {
    const uint64_t threshold = (0 - range) % range;
    while (low < threshold) {
      prod = (unsigned __int128)or_mt64_next(g) * range;
      low = (uint64_t)prod;
    }
  }
  return a + (uint64_t)(prod >> 64);
}

void or_mt64_stream(uint64_t seed, uint64_t count, uint64_t* out) {
  mt64_t g;
  or_mt64_seed(&g, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = or_mt64_next(&g);
}

/* the padding picks j_i = uniform(i, csize-1), i < need (knn_softmax.cpp:45-46) */
void or_uniform_picks(uint64_t seed, uint64_t csize, uint64_t need, uint64_t* out) {
  mt64_t g;
  or_mt64_seed(&g, seed);
  for (uint64_t i = 0; i < need; ++i) out[i] = or_uniform_u64(&g, i, csize - 1);
}

/* ------------------------------------------------------------------------- */
/* ShardLayout, knn_graph.cpp:94-115                                          */
/* ------------------------------------------------------------------------- */
void or_shard_range(uint64_t n, uint64_t p, uint64_t s, uint64_t* begin, uint64_t* end) {
  const uint64_t base = n / p, rem = n % p;
  if (s < rem) {
    *begin = s * (base + 1);
    *end = *begin + base + 1;
  } else {
    *begin = rem * (base + 1) + (s - rem) * base;
    *end = *begin + base;
  }
}

uint64_t or_shard_of(uint64_t n, uint64_t p, uint64_t cls) {
  const uint64_t base = n / p, rem = n % p, big = rem * (base + 1);
  if (cls < big) return cls / (base + 1);
  return rem + (cls - big) / base;
}

/* ------------------------------------------------------------------------- */
/* compress_graph, knn_graph.cpp:235-266.  Output arrays sized by caller:     */
/* k_per_class[n], offsets[n], flat[n*k] (upper bound).  Returns Σ kept.      */
/* ------------------------------------------------------------------------- */
uint64_t or_compress_graph(uint64_t n, uint64_t k, const uint32_t* g_flat, uint64_t p,
                           uint64_t shard, uint32_t* k_per_class, uint64_t* offsets,
                           uint32_t* flat_out) {
  uint64_t begin, end;
  or_shard_range(n, p, shard, &begin, &end);
  uint64_t off = 0;
  for (uint64_t c = 0; c < n; ++c) {
    offsets[c] = off;
    uint32_t kept = 0;
    for (uint64_t r = 0; r < k; ++r) {
      const uint32_t nb = g_flat[c * k + r];
      if (nb >= begin && nb < end) {
        flat_out[off + kept] = nb;
        ++kept;
      }
    }
    k_per_class[c] = kept;
    off += kept;
  }
  return off;
}

/* ------------------------------------------------------------------------- */
/* Active-class selection: select_active_classes (full graph :100-115,        */
/* shards :117-134) + finish_selection (knn_softmax.cpp:17-81).               */
/* The unordered_map pool is restated as dense arrays over [0, N); outputs    */
/* are canonicalised by the reference's final sorts, so iteration order does  */
/* not matter.                                                                */
/* ------------------------------------------------------------------------- */
typedef struct {
  uint32_t cls, best_rank, occ;
} rest_t;

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

static int cmp_rest(const void* pa, const void* pb) { /* knn_softmax.cpp:61-67 */
  const rest_t* a = (const rest_t*)pa;
  const rest_t* b = (const rest_t*)pb;
  if (a->best_rank != b->best_rank) return a->best_rank < b->best_rank ? -1 : 1;
  if (a->occ != b->occ) return a->occ > b->occ ? -1 : 1;
  return (a->cls > b->cls) - (a->cls < b->cls);
}

static int bsearch_u32(const uint32_t* v, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = (lo + hi) / 2;
    if (v[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo < n && v[lo] == x;
}

/* pool given as best_rank[n] (UINT32_MAX = absent) and occ[n]. */
static int finish_selection(uint64_t n, const uint32_t* best_rank, const uint32_t* occ,
                            const uint32_t* labels, uint64_t b, uint64_t m_active, uint64_t seed,
                            uint32_t* out, uint64_t* out_count, int* contains_all) {
  uint32_t* distinct = (uint32_t*)malloc((b ? b : 1) * sizeof(uint32_t));
  memcpy(distinct, labels, b * sizeof(uint32_t));
  qsort(distinct, b, sizeof(uint32_t), cmp_u32);
  uint64_t nd = 0;
  for (uint64_t i = 0; i < b; ++i)
    if (nd == 0 || distinct[nd - 1] != distinct[i]) distinct[nd++] = distinct[i];
  if (m_active < nd) { free(distinct); return OR_ERR_M_TOO_SMALL; }
  if (m_active > n) { free(distinct); return OR_ERR_INVALID_ARGUMENT; }

  uint64_t pool_size = 0;
  for (uint64_t c = 0; c < n; ++c) pool_size += best_rank[c] != UINT32_MAX;

  uint64_t cnt = 0;
  if (pool_size <= m_active) {
    for (uint64_t c = 0; c < n; ++c)
      if (best_rank[c] != UINT32_MAX) out[cnt++] = (uint32_t)c; /* already sorted */
    if (pool_size < m_active) {
      /* complement in ascending order, partial Fisher-Yates (:39-49) */
      const uint64_t csize = n - pool_size;
      uint32_t* comp = (uint32_t*)malloc((csize ? csize : 1) * sizeof(uint32_t));
      uint64_t j = 0;
      for (uint64_t c = 0; c < n; ++c)
        if (best_rank[c] == UINT32_MAX) comp[j++] = (uint32_t)c;
      mt64_t g;
      or_mt64_seed(&g, seed);
      const uint64_t need = m_active - pool_size;
      for (uint64_t i = 0; i < need; ++i) {
        const uint64_t pick = or_uniform_u64(&g, i, csize - 1);
        const uint32_t t = comp[i];
        comp[i] = comp[pick];
        comp[pick] = t;
        out[cnt++] = comp[i];
      }
      free(comp);
      qsort(out, cnt, sizeof(uint32_t), cmp_u32);
    }
  } else {
    /* over-full pool (:52-72) */
    for (uint64_t i = 0; i < nd; ++i) out[cnt++] = distinct[i];
    rest_t* rest = (rest_t*)malloc(pool_size * sizeof(rest_t));
    uint64_t nr = 0;
    for (uint64_t c = 0; c < n; ++c) {
      if (best_rank[c] == UINT32_MAX) continue;
      if (bsearch_u32(distinct, nd, (uint32_t)c)) continue;
      rest[nr].cls = (uint32_t)c;
      rest[nr].best_rank = best_rank[c];
      rest[nr].occ = occ[c];
      ++nr;
    }
    qsort(rest, nr, sizeof(rest_t), cmp_rest);
    const uint64_t take = m_active - nd;
    for (uint64_t i = 0; i < take && i < nr; ++i) out[cnt++] = rest[i].cls;
    free(rest);
    qsort(out, cnt, sizeof(uint32_t), cmp_u32);
  }
  *out_count = cnt;
  int all = 1;
  for (uint64_t i = 0; i < nd; ++i) all &= bsearch_u32(out, cnt, distinct[i]);
  *contains_all = all;
  free(distinct);
  return OR_OK;
}

int or_select_active_full(uint64_t n, uint64_t k, const uint32_t* g_flat, const uint32_t* labels,
                          uint64_t b, uint64_t m_active, uint64_t seed, uint32_t* out,
                          uint64_t* out_count, int* contains_all) {
  uint32_t* best = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* occ = (uint32_t*)calloc(n, sizeof(uint32_t));
  for (uint64_t c = 0; c < n; ++c) best[c] = UINT32_MAX;
  int rc = OR_OK;
  for (uint64_t i = 0; i < b && rc == OR_OK; ++i) {
    const uint32_t y = labels[i];
    if (y >= n) { rc = OR_ERR_LABEL_OUT_OF_RANGE; break; }
    for (uint64_t r = 0; r < k; ++r) {
      const uint32_t c = g_flat[(uint64_t)y * k + r];
      if (r < best[c]) best[c] = (uint32_t)r;
      ++occ[c];
    }
  }
  if (rc == OR_OK)
    rc = finish_selection(n, best, occ, labels, b, m_active, seed, out, out_count, contains_all);
  free(best);
  free(occ);
  return rc;
}

int or_select_active_shards(uint64_t n, uint64_t p, const uint32_t* const* k_per_class,
                            const uint64_t* const* offsets, const uint32_t* const* flat,
                            const uint32_t* labels, uint64_t b, uint64_t m_active, uint64_t seed,
                            uint32_t* out, uint64_t* out_count, int* contains_all) {
  if (p == 0) return OR_ERR_INVALID_ARGUMENT;
  uint32_t* best = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* occ = (uint32_t*)calloc(n, sizeof(uint32_t));
  for (uint64_t c = 0; c < n; ++c) best[c] = UINT32_MAX;
  int rc = OR_OK;
  for (uint64_t i = 0; i < b && rc == OR_OK; ++i) {
    const uint32_t y = labels[i];
    if (y >= n) { rc = OR_ERR_LABEL_OUT_OF_RANGE; break; }
    for (uint64_t s = 0; s < p; ++s) {
      const uint32_t kk = k_per_class[s][y];
      const uint32_t* sl = flat[s] + offsets[s][y];
      for (uint32_t r = 0; r < kk; ++r) {
        const uint32_t c = sl[r];
        if (r < best[c]) best[c] = r;
        ++occ[c];
      }
    }
  }
  if (rc == OR_OK)
    rc = finish_selection(n, best, occ, labels, b, m_active, seed, out, out_count, contains_all);
  free(best);
  free(occ);
  return rc;
}

/* select_active_classes(span<CompressedKnnGraph>) with the padding draw's raw mt19937_64 words
 * replaced by words[0..nwords) (words past the end read as 0): drives the Lemire rejection loop
 * of uniform_int_distribution (uniform_int_dist.h:268-272) deterministically -- a zero word is
 * always rejected unless the range is a power of two.  Not thread-safe (test hook). */
int or_select_active_shards_stream(uint64_t n, uint64_t p, const uint32_t* const* k_per_class,
                                   const uint64_t* const* offsets, const uint32_t* const* flat,
                                   const uint32_t* labels, uint64_t b, uint64_t m_active,
                                   const uint64_t* words, uint64_t nwords, uint32_t* out,
                                   uint64_t* out_count, int* contains_all) {
  g_inj_words = words;
  g_inj_len = nwords;
  const int rc = or_select_active_shards(n, p, k_per_class, offsets, flat, labels, b, m_active, 0,
                                         out, out_count, contains_all);
  g_inj_words = NULL;
  g_inj_len = 0;
  return rc;
}

/* ------------------------------------------------------------------------- */
/* Core math, matrix.cpp                                                      */
/* ------------------------------------------------------------------------- */

/* l2_normalize_rows_cached, matrix.cpp:12-29.  Returns OR_OK or -(1+row)    */
/* encoded through *bad_row with OR_ERR_ZERO_NORM_ROW.                        */
int or_l2_normalize_rows(uint64_t rows, uint64_t cols, const float* in, float eps, float* out,
                         float* norms, uint64_t* bad_row) {
  if (rows == 0 || cols == 0) return OR_ERR_SHAPE_MISMATCH;
  for (uint64_t i = 0; i < rows; ++i) {
    const float* src = in + i * cols;
    double sq = 0.0;
    for (uint64_t j = 0; j < cols; ++j) sq += (double)src[j] * src[j];
    const float norm = (float)sqrt(sq);
    if (norm < eps) { *bad_row = i; return OR_ERR_ZERO_NORM_ROW; }
    norms[i] = norm;
    float* dst = out + i * cols;
    const float inv = 1.0f / norm;
    for (uint64_t j = 0; j < cols; ++j) dst[j] = src[j] * inv;
  }
  return OR_OK;
}

/* l2_normalize_backward, matrix.cpp:31-48 (also the inline W version,       */
/* parallel.cpp:653-666, which is the same arithmetic per row).               */
void or_l2_normalize_backward(uint64_t rows, uint64_t cols, const float* nrm, const float* norms,
                              const float* g_in, float* g_out) {
  for (uint64_t i = 0; i < rows; ++i) {
    const float* nh = nrm + i * cols;
    const float* g = g_in + i * cols;
    double dot = 0.0;
    for (uint64_t j = 0; j < cols; ++j) dot += (double)g[j] * nh[j];
    const float d = (float)dot;
    const float inv = 1.0f / norms[i];
    float* o = g_out + i * cols;
    for (uint64_t j = 0; j < cols; ++j) o[j] = (g[j] - d * nh[j]) * inv;
  }
}

/* The three matmuls below are parallelised over OUTPUT elements with OpenMP (each thread owns
 * whole output rows / columns and runs the reference's per-element chain unchanged), so their
 * results are bit-identical to the sequential loops of matrix.cpp at any thread count. */

/* matmul(a, b, transpose_b=true), matrix.cpp:57-68: c = a·bᵀ, ascending k.  Four output columns
 * are advanced together (independent chains, each in ascending k). */
void or_matmul_nt(uint64_t m, uint64_t n, uint64_t kd, const float* a, const float* b, float* c) {
#pragma omp parallel for schedule(dynamic, 1) if (m * n * kd > (1u << 22))
  for (uint64_t i = 0; i < m; ++i) {
    const float* ai = a + i * kd;
    uint64_t j = 0;
    for (; j + 4 <= n; j += 4) {
      const float *b0 = b + j * kd, *b1 = b0 + kd, *b2 = b1 + kd, *b3 = b2 + kd;
      float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
      for (uint64_t k = 0; k < kd; ++k) {
        const float x = ai[k];
        a0 += x * b0[k];
        a1 += x * b1[k];
        a2 += x * b2[k];
        a3 += x * b3[k];
      }
      c[i * n + j] = a0;
      c[i * n + j + 1] = a1;
      c[i * n + j + 2] = a2;
      c[i * n + j + 3] = a3;
    }
    for (; j < n; ++j) {
      const float* bj = b + j * kd;
      float acc = 0.0f;
      for (uint64_t k = 0; k < kd; ++k) acc += ai[k] * bj[k];
      c[i * n + j] = acc;
    }
  }
}

/* matmul(a, b) (ikj), matrix.cpp:69-80: c[m×n] = a[m×kd]·b[kd×n] */
void or_matmul_nn(uint64_t m, uint64_t n, uint64_t kd, const float* a, const float* b, float* c) {
  memset(c, 0, m * n * sizeof(float));
#pragma omp parallel for schedule(dynamic, 1) if (m * n * kd > (1u << 22))
  for (uint64_t i = 0; i < m; ++i) {
    const float* ai = a + i * kd;
    float* ci = c + i * n;
    for (uint64_t k = 0; k < kd; ++k) {
      const float aik = ai[k];
      const float* bk = b + k * n;
      for (uint64_t j = 0; j < n; ++j) ci[j] += aik * bk[j];
    }
  }
}

/* matmul_at(a, b), matrix.cpp:84-98: c[ac×bc] = aᵀ·b, ascending i (every c[j][l] accumulates
 * rows i = 0, 1, ... in order; threads own blocks of output rows j) */
void or_matmul_tn(uint64_t rows, uint64_t ac, uint64_t bc, const float* a, const float* b, float* c) {
  memset(c, 0, ac * bc * sizeof(float));
  const uint64_t JB = 64;
#pragma omp parallel for schedule(dynamic, 1) if (rows * ac * bc > (1u << 22))
  for (uint64_t j0 = 0; j0 < ac; j0 += JB) {
    const uint64_t j1 = j0 + JB < ac ? j0 + JB : ac;
    for (uint64_t i = 0; i < rows; ++i) {
      const float* ai = a + i * ac;
      const float* bi = b + i * bc;
      for (uint64_t j = j0; j < j1; ++j) {
        const float aij = ai[j];
        float* cj = c + j * bc;
        for (uint64_t l = 0; l < bc; ++l) cj[l] += aij * bi[l];
      }
    }
  }
}

/* ------------------------------------------------------------------------- */
/* softmax_xent, softmax.cpp:8-39                                             */
/* ------------------------------------------------------------------------- */
int or_softmax_xent(uint64_t m, uint64_t c, const float* logits, const uint32_t* labels,
                    double* loss, float* grad) {
  for (uint64_t i = 0; i < m; ++i)
    if (labels[i] >= c) return OR_ERR_LABEL_OUT_OF_RANGE;
  const float inv_m = 1.0f / (float)m;
  double loss_sum = 0.0;
  for (uint64_t i = 0; i < m; ++i) {
    const float* row = logits + i * c;
    float* grow = grad + i * c;
    float maxv = row[0];
    for (uint64_t j = 1; j < c; ++j) maxv = maxv < row[j] ? row[j] : maxv; /* std::max */
    double denom = 0.0;
    for (uint64_t j = 0; j < c; ++j) {
      const float e = expf(row[j] - maxv);
      grow[j] = e;
      denom += e;
    }
    const float inv_denom = (float)(1.0 / denom);
    for (uint64_t j = 0; j < c; ++j) grow[j] = grow[j] * inv_denom * inv_m;
    grow[labels[i]] -= inv_m;
    loss_sum += log(denom) - (double)(row[labels[i]] - maxv);
  }
  *loss = loss_sum / (double)m;
  return OR_OK;
}

/* knn_softmax_forward_backward, knn_softmax.cpp:136-186: gather of the active rows of w_norm
 * (LabelOutOfRange for an id >= n), labels remapped by position_of (LabelNotActive), logits =
 * matmul(x, w_active, T) then *= scale, softmax_xent, grad_features = matmul(G, w_active) *
 * scale, grad_weights[active[i]] = matmul_at(G, x)[i] * scale (returned compact: m_act x d). */
int or_knn_softmax_forward_backward(uint64_t b, uint64_t n, uint64_t d, const float* x,
                                    const float* w, const uint32_t* labels, const uint32_t* active,
                                    uint64_t m_act, float scale, double* loss, float* grad_logits,
                                    float* grad_features, float* grad_w_active) {
  if (m_act == 0) return OR_ERR_INVALID_ARGUMENT;
  float* wa = (float*)malloc(m_act * d * sizeof(float));
  uint32_t* rl = (uint32_t*)malloc((b ? b : 1) * sizeof(uint32_t));
  int rc = OR_OK;
  for (uint64_t i = 0; i < m_act && rc == OR_OK; ++i) {
    if (active[i] >= n) rc = OR_ERR_LABEL_OUT_OF_RANGE;
    else memcpy(wa + i * d, w + (uint64_t)active[i] * d, d * sizeof(float));
  }
  for (uint64_t i = 0; i < b && rc == OR_OK; ++i) {
    uint64_t lo = 0, hi = m_act; /* ActiveSet::position_of, lower_bound */
    while (lo < hi) { uint64_t mid = (lo + hi) / 2; if (active[mid] < labels[i]) lo = mid + 1; else hi = mid; }
    if (lo == m_act || active[lo] != labels[i]) rc = OR_ERR_LABEL_NOT_ACTIVE;
    else rl[i] = (uint32_t)lo;
  }
  if (rc == OR_OK) {
    float* lg = (float*)malloc(b * m_act * sizeof(float));
    or_matmul_nt(b, m_act, d, x, wa, lg);
    for (uint64_t t = 0; t < b * m_act; ++t) lg[t] *= scale;
    rc = or_softmax_xent(b, m_act, lg, rl, loss, grad_logits);
    free(lg);
  }
  if (rc == OR_OK) {
    or_matmul_nn(b, d, m_act, grad_logits, wa, grad_features);
    for (uint64_t t = 0; t < b * d; ++t) grad_features[t] *= scale;
    or_matmul_tn(b, m_act, d, grad_logits, x, grad_w_active);
    for (uint64_t t = 0; t < m_act * d; ++t) grad_w_active[t] = grad_w_active[t] * scale;
  }
  free(wa);
  free(rl);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* distributed_softmax_xent_cols, parallel.cpp:106-188 (rank-ordered          */
/* scalar_reduce :66-88).  logits[s] is m × ncols[s]; cols[s] sorted ids.     */
/* ------------------------------------------------------------------------- */
int or_distributed_softmax_xent_cols(uint64_t p, uint64_t m, const float* const* logits,
                                     const uint32_t* const* cols, const uint64_t* ncols,
                                     const uint32_t* labels, double* loss, float* const* grads) {
  double* gmax = (double*)malloc(m * sizeof(double));
  double* sums = (double*)calloc(3 * m, sizeof(double));
  double* local = (double*)malloc(3 * m * sizeof(double));
  for (uint64_t s = 0; s < p; ++s) {
    for (uint64_t i = 0; i < m; ++i) {
      const float* row = logits[s] + i * ncols[s];
      float mx = ncols[s] ? row[0] : -INFINITY;
      for (uint64_t j = 1; j < ncols[s]; ++j) mx = mx < row[j] ? row[j] : mx;
      const double v = (double)mx;
      if (s == 0) gmax[i] = v;
      else gmax[i] = gmax[i] < v ? v : gmax[i]; /* std::max(out, in) */
    }
  }
  for (uint64_t s = 0; s < p; ++s) {
    memset(local, 0, 3 * m * sizeof(double));
    for (uint64_t i = 0; i < m; ++i) {
      const float* row = logits[s] + i * ncols[s];
      const float mx = (float)gmax[i];
      double denom = 0.0;
      for (uint64_t j = 0; j < ncols[s]; ++j) denom += expf(row[j] - mx);
      local[i] = denom;
      uint64_t lo = 0, hi = ncols[s];
      while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (cols[s][mid] < labels[i]) lo = mid + 1; else hi = mid;
      }
      if (lo < ncols[s] && cols[s][lo] == labels[i]) {
        local[m + i] = (double)(row[lo] - mx);
        local[2 * m + i] = 1.0;
      }
    }
    for (uint64_t i = 0; i < 3 * m; ++i) {
      if (s == 0) sums[i] = local[i];
      else sums[i] += local[i];
    }
  }
  int rc = OR_OK;
  for (uint64_t i = 0; i < m; ++i)
    if (sums[2 * m + i] != 1.0) rc = OR_ERR_LABEL_OUT_OF_RANGE;
  if (rc == OR_OK) {
    double loss_sum = 0.0;
    for (uint64_t i = 0; i < m; ++i) loss_sum += log(sums[i]) - sums[m + i];
    *loss = loss_sum / (double)m;
    const float inv_m = 1.0f / (float)m;
    for (uint64_t s = 0; s < p; ++s) {
      for (uint64_t i = 0; i < m; ++i) {
        const float* row = logits[s] + i * ncols[s];
        float* grow = grads[s] + i * ncols[s];
        const float mx = (float)gmax[i];
        const float inv_denom = (float)(1.0 / sums[i]);
        for (uint64_t j = 0; j < ncols[s]; ++j) grow[j] = expf(row[j] - mx) * inv_denom * inv_m;
        uint64_t lo = 0, hi = ncols[s];
        while (lo < hi) {
          uint64_t mid = (lo + hi) / 2;
          if (cols[s][mid] < labels[i]) lo = mid + 1; else hi = mid;
        }
        if (lo < ncols[s] && cols[s][lo] == labels[i]) grow[lo] -= inv_m;
      }
    }
  }
  free(gmax);
  free(sums);
  free(local);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* SgdMomentum::step_rows, fccs.cpp:74-89 (velocity given, dense n_rows×cols) */
/* ------------------------------------------------------------------------- */
void or_sgd_step_rows(uint64_t cols, float* params, const float* grad_rows, float* velocity,
                      const uint32_t* rows, uint64_t nrows, float lr, float momentum, float wd) {
  for (uint64_t t = 0; t < nrows; ++t) {
    const uint64_t r = rows[t];
    float* p = params + r * cols;
    const float* g = grad_rows + t * cols; /* compact: one grad row per listed row */
    float* vel = velocity + r * cols;
    for (uint64_t j = 0; j < cols; ++j) {
      const float v = momentum * vel[j] + g[j] + wd * p[j];
      vel[j] = v;
      p[j] -= lr * v;
    }
  }
}

/* ------------------------------------------------------------------------- */
/* build_graph_bruteforce, knn_graph.cpp:124-145 with CandidateList::offer    */
/* (:35-43) and better (:20-26).  Exact top-k under (self, score↓, idx↑).    */
/* ------------------------------------------------------------------------- */
static int better(float sa, uint32_t ia, float sb, uint32_t ib, uint32_t self) {
  const int as = ia == self, bs = ib == self;
  if (as != bs) return as;
  if (sa != sb) return sa > sb;
  return ia < ib;
}

int or_build_graph_bruteforce(uint64_t n, uint64_t d, const float* w, uint64_t k, uint32_t* out) {
  if (k > n) return OR_ERR_K_TOO_LARGE;
  if (k == 0) return OR_ERR_INVALID_ARGUMENT;
  float* sc = (float*)malloc(k * sizeof(float));
  uint32_t* ix = (uint32_t*)malloc(k * sizeof(uint32_t));
  for (uint64_t j = 0; j < n; ++j) {
    uint64_t sz = 0;
    const float* wj = w + j * d;
    for (uint64_t i = 0; i < n; ++i) {
      const float* wi = w + i * d;
      float dot = 0.0f;
      for (uint64_t t = 0; t < d; ++t) dot += wj[t] * wi[t];
      if (sz == k && !better(dot, (uint32_t)i, sc[sz - 1], ix[sz - 1], (uint32_t)j)) continue;
      uint64_t pos = 0; /* lower_bound under better */
      while (pos < sz && better(sc[pos], ix[pos], dot, (uint32_t)i, (uint32_t)j)) ++pos;
      uint64_t last = sz < k ? sz : k - 1;
      for (uint64_t q = last; q > pos; --q) { sc[q] = sc[q - 1]; ix[q] = ix[q - 1]; }
      sc[pos] = dot;
      ix[pos] = (uint32_t)i;
      if (sz < k) ++sz;
    }
    memcpy(out + j * k, ix, k * sizeof(uint32_t));
  }
  free(sc);
  free(ix);
  return OR_OK;
}

/* One row of build_graph_bruteforce: the exact k neighbours of class j (same arithmetic and
   ordering), for sampled-row checks at sizes where the full O(N^2 D) oracle is too slow. */
int or_graph_row(uint64_t n, uint64_t d, const float* w, uint64_t j, uint64_t k, uint32_t* out) {
  if (k > n) return OR_ERR_K_TOO_LARGE;
  if (k == 0) return OR_ERR_INVALID_ARGUMENT;
  float* sc = (float*)malloc(k * sizeof(float));
  uint32_t* ix = (uint32_t*)malloc(k * sizeof(uint32_t));
  uint64_t sz = 0;
  const float* wj = w + j * d;
  for (uint64_t i = 0; i < n; ++i) {
    const float* wi = w + i * d;
    float dot = 0.0f;
    for (uint64_t t = 0; t < d; ++t) dot += wj[t] * wi[t];
    if (sz == k && !better(dot, (uint32_t)i, sc[sz - 1], ix[sz - 1], (uint32_t)j)) continue;
    uint64_t pos = 0;
    while (pos < sz && better(sc[pos], ix[pos], dot, (uint32_t)i, (uint32_t)j)) ++pos;
    uint64_t last = sz < k ? sz : k - 1;
    for (uint64_t q = last; q > pos; --q) { sc[q] = sc[q - 1]; ix[q] = ix[q - 1]; }
    sc[pos] = dot;
    ix[pos] = (uint32_t)i;
    if (sz < k) ++sz;
  }
  memcpy(out, ix, k * sizeof(uint32_t));
  free(sc);
  free(ix);
  return OR_OK;
}

/* Sampled rows of build_graph_bruteforce over a class matrix streamed in chunks (for checks at
   sizes where the matrix does not fit host memory): nq query rows (global ids qid[], vectors q)
   keep their exact top-k lists (sc/ix/sz, nq x k) under `better` while chunks of rows
   [base, base + rows) pass by, in any order -- `better` is a strict total order, so the final
   lists equal or_graph_row's.  Same per-pair arithmetic as or_graph_row (ascending-d fp32 dot).
   Parallel over row blocks of the chunk (private lists, merged under the same order). */
static void cand_insert(float* sc, uint32_t* ix, uint64_t* sz, uint64_t k, float dot, uint32_t i,
                        uint32_t self) {
  if (*sz == k && !better(dot, i, sc[*sz - 1], ix[*sz - 1], self)) return;
  uint64_t pos = 0;
  while (pos < *sz && better(sc[pos], ix[pos], dot, i, self)) ++pos;
  uint64_t last = *sz < k ? *sz : k - 1;
  for (uint64_t q = last; q > pos; --q) { sc[q] = sc[q - 1]; ix[q] = ix[q - 1]; }
  sc[pos] = dot;
  ix[pos] = i;
  if (*sz < k) ++*sz;
}

void or_graph_rows_update(uint64_t nq, uint64_t d, const float* q, const uint64_t* qid, uint64_t k,
                          const float* chunk, uint64_t rows, uint64_t base, float* sc, uint32_t* ix,
                          uint64_t* sz) {
  const uint64_t RB = 4096, nb = (rows + RB - 1) / RB;
  float* psc = (float*)malloc(nb * nq * k * sizeof(float));
  uint32_t* pix = (uint32_t*)malloc(nb * nq * k * sizeof(uint32_t));
  uint64_t* psz = (uint64_t*)calloc(nb * nq, sizeof(uint64_t));
#pragma omp parallel for schedule(dynamic, 1)
  for (uint64_t blk = 0; blk < nb; ++blk) {
    const uint64_t r1 = (blk + 1) * RB < rows ? (blk + 1) * RB : rows;
    for (uint64_t r = blk * RB; r < r1; ++r) {
      const float* wi = chunk + r * d;
      for (uint64_t a = 0; a < nq; ++a) {
        const float* wj = q + a * d;
        float dot = 0.0f;
        for (uint64_t t = 0; t < d; ++t) dot += wj[t] * wi[t];
        const uint64_t o = blk * nq + a;
        cand_insert(psc + o * k, pix + o * k, psz + o, k, dot, (uint32_t)(base + r),
                    (uint32_t)qid[a]);
      }
    }
  }
  for (uint64_t blk = 0; blk < nb; ++blk)
    for (uint64_t a = 0; a < nq; ++a) {
      const uint64_t o = blk * nq + a;
      for (uint64_t e = 0; e < psz[o]; ++e)
        cand_insert(sc + a * k, ix + a * k, sz + a, k, psc[o * k + e], pix[o * k + e],
                    (uint32_t)qid[a]);
    }
  free(psc);
  free(pix);
  free(psz);
}

/* classify_retrieval (the reference tree has no implementation, this
   restates the spec): the nearest class of each query among the L2-normalized class weights,
   i.e. the argmax of the cosine logits matmul(q_hat, w_hat, T) (matrix.cpp:57-68 order; the
   logit scale does not move the argmax), ties to the lower class index.  q and w are
   normalized with l2_normalize_rows (matrix.cpp:12-29).  out_score: the winning cosine. */
int or_classify_retrieval(uint64_t nq, uint64_t n, uint64_t d, const float* q, const float* w,
                          uint32_t* out_class, float* out_score) {
  if (nq == 0 || n == 0 || d == 0) return OR_ERR_SHAPE_MISMATCH;
  float* qn = (float*)malloc(nq * d * sizeof(float));
  float* wn = (float*)malloc(n * d * sizeof(float));
  float* nq_norm = (float*)malloc(nq * sizeof(float));
  float* nw_norm = (float*)malloc(n * sizeof(float));
  uint64_t bad = 0;
  int rc = or_l2_normalize_rows(nq, d, q, 1e-12f, qn, nq_norm, &bad);
  if (rc == OR_OK) rc = or_l2_normalize_rows(n, d, w, 1e-12f, wn, nw_norm, &bad);
  for (uint64_t i = 0; rc == OR_OK && i < nq; ++i) {
    const float* qi = qn + i * d;
    float best = 0.0f;
    uint32_t arg = 0;
    for (uint64_t j = 0; j < n; ++j) {
      const float* wj = wn + j * d;
      float acc = 0.0f;
      for (uint64_t t = 0; t < d; ++t) acc += qi[t] * wj[t];
      if (j == 0 || acc > best) {
        best = acc;
        arg = (uint32_t)j;
      }
    }
    out_class[i] = arg;
    if (out_score) out_score[i] = best;
  }
  free(qn);
  free(wn);
  free(nq_norm);
  free(nw_norm);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* The fc half of HybridSim::train_step in kKnn mode with one micro-batch    */
/* (parallel.cpp:455-572, :638-668), the composite the device layer replaces. */
/*                                                                            */
/* Inputs: W (n × d, all shards concatenated), velocity (n × d, updated in    */
/* place, zeros on the first step as ensure_state does), the global batch of  */
/* already-extracted features x (b × d, rank-major), labels, per-shard CSR    */
/* graphs.  Outputs: loss, active set, grad_feat (b × d) = gradient w.r.t.    */
/* the raw features (the tensor handed to mlp_backward, :585-586).            */
/* ------------------------------------------------------------------------- */
int or_fc_train_step(uint64_t n, uint64_t d, uint64_t p, float* w, float* velocity,
                     const float* x, const uint32_t* labels, uint64_t b,
                     const uint32_t* const* k_per_class, const uint64_t* const* offsets,
                     const uint32_t* const* flat, uint64_t m_active, uint64_t seed, float scale,
                     float lr, float momentum, float wd, double* loss_out, uint32_t* active_out,
                     uint64_t* active_count, float* grad_feat, float* logits_out) {
  if (b == 0 || b % p != 0) return OR_ERR_INVALID_ARGUMENT;
  for (uint64_t i = 0; i < b; ++i)
    if (labels[i] >= n) return OR_ERR_LABEL_OUT_OF_RANGE;
  int contains_all = 0;
  int rc = or_select_active_shards(n, p, k_per_class, offsets, flat, labels, b, m_active, seed,
                                   active_out, active_count, &contains_all);
  if (rc != OR_OK) return rc;
  const uint64_t na = *active_count;

  /* worker_cols (:479-486) */
  uint64_t* lo = (uint64_t*)malloc((p + 1) * sizeof(uint64_t));
  for (uint64_t s = 0; s <= p; ++s) {
    uint64_t bg, en;
    if (s < p) or_shard_range(n, p, s, &bg, &en); else bg = n;
    uint64_t a = 0, z = na;
    while (a < z) { uint64_t mid = (a + z) / 2; if (active_out[mid] < bg) a = mid + 1; else z = mid; }
    lo[s] = a;
  }

  /* normalized active rows (row-wise identical to normalizing the shard) */
  float* wsub = (float*)malloc((na ? na : 1) * d * sizeof(float));
  float* wnorm = (float*)malloc((na ? na : 1) * sizeof(float));
  for (uint64_t i = 0; i < na; ++i) {
    uint64_t bad;
    rc = or_l2_normalize_rows(1, d, w + (uint64_t)active_out[i] * d, 1e-12f, wsub + i * d,
                              wnorm + i, &bad);
    if (rc != OR_OK) { rc = OR_ERR_ZERO_NORM_ROW; goto out_w; }
  }
  float* fhat = (float*)malloc(b * d * sizeof(float));
  float* fnorm = (float*)malloc(b * sizeof(float));
  {
    uint64_t bad;
    rc = or_l2_normalize_rows(b, d, x, 1e-12f, fhat, fnorm, &bad);
  }
  if (rc != OR_OK) goto out_f;

  {
    const float** lg = (const float**)malloc(p * sizeof(float*));
    float** gr = (float**)malloc(p * sizeof(float*));
    const uint32_t** cl = (const uint32_t**)malloc(p * sizeof(uint32_t*));
    uint64_t* nc = (uint64_t*)malloc(p * sizeof(uint64_t));
    for (uint64_t s = 0; s < p; ++s) {
      nc[s] = lo[s + 1] - lo[s];
      cl[s] = active_out + lo[s];
      float* l = (float*)malloc((nc[s] ? nc[s] : 1) * b * sizeof(float));
      or_matmul_nt(b, nc[s], d, fhat, wsub + lo[s] * d, l);
      for (uint64_t t = 0; t < b * nc[s]; ++t) l[t] *= scale; /* :551 */
      lg[s] = l;
      gr[s] = (float*)malloc((nc[s] ? nc[s] : 1) * b * sizeof(float));
    }
    if (logits_out) /* concatenated in active order: rank-major == sorted */
      for (uint64_t s = 0; s < p; ++s)
        for (uint64_t i = 0; i < b; ++i)
          memcpy(logits_out + i * na + lo[s], lg[s] + i * nc[s], nc[s] * sizeof(float));
    double loss = 0.0;
    rc = or_distributed_softmax_xent_cols(p, b, lg, cl, nc, labels, &loss, gr);
    if (rc == OR_OK) {
      *loss_out = 0.0 + (double)1.0f * loss; /* :558, weight = 1 */
      float* fsum = (float*)calloc(b * d, sizeof(float));
      float* tmp = (float*)malloc(b * d * sizeof(float));
      for (uint64_t s = 0; s < p; ++s) {
        /* weight side (:564-566): gw = matmul_at(G, f̂) · (scale·weight) */
        float* gw = (float*)malloc((nc[s] ? nc[s] : 1) * d * sizeof(float));
        or_matmul_tn(b, nc[s], d, gr[s], fhat, gw);
        const float sw = scale * 1.0f;
        for (uint64_t t = 0; t < nc[s] * d; ++t) gw[t] *= sw;
        for (uint64_t t = 0; t < nc[s] * d; ++t) gw[t] = 0.0f + 1.0f * gw[t]; /* axpy into fc_acc */
        /* normalize-backward + step_rows on the active rows (:649-667) */
        float* graw = (float*)malloc((nc[s] ? nc[s] : 1) * d * sizeof(float));
        or_l2_normalize_backward(nc[s], d, wsub + lo[s] * d, wnorm + lo[s], gw, graw);
        or_sgd_step_rows(d, w, graw, velocity, active_out + lo[s], nc[s], lr, momentum, wd);
        free(graw);
        free(gw);
        /* feature side (:568-569) and the rank-order all_reduce_sum (:572) */
        or_matmul_nn(b, d, nc[s], gr[s], wsub + lo[s] * d, tmp);
        for (uint64_t t = 0; t < b * d; ++t) tmp[t] *= scale;
        if (s == 0) memcpy(fsum, tmp, b * d * sizeof(float));
        else for (uint64_t t = 0; t < b * d; ++t) fsum[t] += 1.0f * tmp[t];
      }
      /* feature normalize-backward (:574-585) */
      or_l2_normalize_backward(b, d, fhat, fnorm, fsum, grad_feat);
      free(fsum);
      free(tmp);
    }
    for (uint64_t s = 0; s < p; ++s) { free((void*)lg[s]); free(gr[s]); }
    free(lg); free(gr); free(cl); free(nc);
  }
out_f:
  free(fhat);
  free(fnorm);
out_w:
  free(wsub);
  free(wnorm);
  free(lo);
  return rc;
}

/* The fc half of HybridSim::train_step with `micro_batches` micro-batches (parallel.cpp:444,
 * :505-591, :638-668): one selection and one normalized W_sub per step; per micro-batch c
 * (balanced split of every worker's slice, :514-523) the rank-major micro batch of m_c = rows_c*p
 * rows gets its own logits, distributed softmax (G carries 1/m_c), loss weighted by
 * weight_c = float(m_c)/float(m) (:553-558), weight-side gradient scaled by scale*weight_c and
 * accumulated into fc_acc with axpy (:564-566), and feature gradient (:568-585).  The update
 * runs once, after the last micro-batch (:638-668).  grad_feat row i of worker w's slice is the
 * gradient handed to mlp_backward for that row (micro-scaled: 1/m_c, not 1/m). */
int or_fc_train_step_mb(uint64_t n, uint64_t d, uint64_t p, float* w, float* velocity,
                        const float* x, const uint32_t* labels, uint64_t b,
                        const uint32_t* const* k_per_class, const uint64_t* const* offsets,
                        const uint32_t* const* flat, uint64_t m_active, uint64_t seed,
                        float scale, float lr, float momentum, float wd, uint64_t micro_batches,
                        double* loss_out, uint32_t* active_out, uint64_t* active_count,
                        float* grad_feat) {
  if (b == 0 || b % p != 0) return OR_ERR_INVALID_ARGUMENT;
  for (uint64_t i = 0; i < b; ++i)
    if (labels[i] >= n) return OR_ERR_LABEL_OUT_OF_RANGE;
  const uint64_t slice = b / p;
  uint64_t micros = micro_batches ? micro_batches : 1;
  if (micros > slice) micros = slice;
  int contains_all = 0;
  int rc = or_select_active_shards(n, p, k_per_class, offsets, flat, labels, b, m_active, seed,
                                   active_out, active_count, &contains_all);
  if (rc != OR_OK) return rc;
  const uint64_t na = *active_count;
  uint64_t* lo = (uint64_t*)malloc((p + 1) * sizeof(uint64_t));
  for (uint64_t s = 0; s <= p; ++s) {
    uint64_t bg, en;
    if (s < p) or_shard_range(n, p, s, &bg, &en); else bg = n;
    uint64_t a = 0, z = na;
    while (a < z) { uint64_t mid = (a + z) / 2; if (active_out[mid] < bg) a = mid + 1; else z = mid; }
    lo[s] = a;
  }
  float* wsub = (float*)malloc((na ? na : 1) * d * sizeof(float));
  float* wnorm = (float*)malloc((na ? na : 1) * sizeof(float));
  float* fc_acc = (float*)calloc((na ? na : 1) * d, sizeof(float));
  float* xm = (float*)malloc(b * d * sizeof(float));
  float* fhat = (float*)malloc(b * d * sizeof(float));
  float* fnorm = (float*)malloc(b * sizeof(float));
  uint32_t* lab_m = (uint32_t*)malloc(b * sizeof(uint32_t));
  float* fsum = (float*)malloc(b * d * sizeof(float));
  float* tmp = (float*)malloc(b * d * sizeof(float));
  float* gfm = (float*)malloc(b * d * sizeof(float));
  for (uint64_t i = 0; i < na; ++i) {
    uint64_t bad;
    if (or_l2_normalize_rows(1, d, w + (uint64_t)active_out[i] * d, 1e-12f, wsub + i * d,
                             wnorm + i, &bad) != OR_OK) { rc = OR_ERR_ZERO_NORM_ROW; goto out; }
  }
  {
    double loss_sum = 0.0;
    const uint64_t base = slice / micros, rem = slice % micros;
    uint64_t off = 0;
    for (uint64_t c = 0; c < micros && rc == OR_OK; ++c) {
      const uint64_t rows_c = base + (c < rem ? 1 : 0), mm = rows_c * p;
      const float weight = (float)mm / (float)b;
      for (uint64_t wk = 0; wk < p; ++wk)
        for (uint64_t i = 0; i < rows_c; ++i) {
          lab_m[wk * rows_c + i] = labels[wk * slice + off + i];
          memcpy(xm + (wk * rows_c + i) * d, x + (wk * slice + off + i) * d, d * sizeof(float));
        }
      uint64_t bad;
      rc = or_l2_normalize_rows(mm, d, xm, 1e-12f, fhat, fnorm, &bad);
      if (rc != OR_OK) break;
      const float** lg = (const float**)malloc(p * sizeof(float*));
      float** gr = (float**)malloc(p * sizeof(float*));
      const uint32_t** cl = (const uint32_t**)malloc(p * sizeof(uint32_t*));
      uint64_t* nc = (uint64_t*)malloc(p * sizeof(uint64_t));
      for (uint64_t s = 0; s < p; ++s) {
        nc[s] = lo[s + 1] - lo[s];
        cl[s] = active_out + lo[s];
        float* l = (float*)malloc((nc[s] ? nc[s] : 1) * mm * sizeof(float));
        or_matmul_nt(mm, nc[s], d, fhat, wsub + lo[s] * d, l);
        for (uint64_t t = 0; t < mm * nc[s]; ++t) l[t] *= scale; /* :551 */
        lg[s] = l;
        gr[s] = (float*)malloc((nc[s] ? nc[s] : 1) * mm * sizeof(float));
      }
      double loss = 0.0;
      rc = or_distributed_softmax_xent_cols(p, mm, lg, cl, nc, lab_m, &loss, gr);
      if (rc == OR_OK) {
        loss_sum += (double)weight * loss; /* :558 */
        for (uint64_t s = 0; s < p; ++s) {
          float* gw = (float*)malloc((nc[s] ? nc[s] : 1) * d * sizeof(float));
          or_matmul_tn(mm, nc[s], d, gr[s], fhat, gw);
          const float sw = scale * weight; /* :565 */
          for (uint64_t t = 0; t < nc[s] * d; ++t) gw[t] *= sw;
          float* acc = fc_acc + lo[s] * d;
          for (uint64_t t = 0; t < nc[s] * d; ++t) acc[t] += 1.0f * gw[t]; /* axpy :566 */
          free(gw);
          or_matmul_nn(mm, d, nc[s], gr[s], wsub + lo[s] * d, tmp); /* :568-569 */
          for (uint64_t t = 0; t < mm * d; ++t) tmp[t] *= scale;
          if (s == 0) memcpy(fsum, tmp, mm * d * sizeof(float));
          else for (uint64_t t = 0; t < mm * d; ++t) fsum[t] += 1.0f * tmp[t]; /* :572 */
        }
        /* each worker's own rows back through the normalization (:574-585) */
        or_l2_normalize_backward(mm, d, fhat, fnorm, fsum, gfm);
        for (uint64_t wk = 0; wk < p; ++wk)
          for (uint64_t i = 0; i < rows_c; ++i)
            memcpy(grad_feat + (wk * slice + off + i) * d, gfm + (wk * rows_c + i) * d,
                   d * sizeof(float));
      }
      for (uint64_t s = 0; s < p; ++s) { free((void*)lg[s]); free(gr[s]); }
      free(lg); free(gr); free(cl); free(nc);
      off += rows_c;
    }
    if (rc == OR_OK) {
      *loss_out = loss_sum;
      /* the update, once (:638-668) */
      float* graw = (float*)malloc((na ? na : 1) * d * sizeof(float));
      for (uint64_t s = 0; s < p; ++s) {
        const uint64_t ns = lo[s + 1] - lo[s];
        or_l2_normalize_backward(ns, d, wsub + lo[s] * d, wnorm + lo[s], fc_acc + lo[s] * d,
                                 graw);
        or_sgd_step_rows(d, w, graw, velocity, active_out + lo[s], ns, lr, momentum, wd);
      }
      free(graw);
    }
  }
out:
  free(lo); free(wsub); free(wnorm); free(fc_acc); free(xm); free(fhat); free(fnorm);
  free(lab_m); free(fsum); free(tmp); free(gfm);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* DGC sparsification (sparsify.cpp), beside the fc path                      */
/* ------------------------------------------------------------------------- */

typedef struct {
  float v;
  uint64_t i;
} OrEntry;

/* `precedes` (sparsify.cpp:19-24): |value| descending, index ascending */
static int or_precedes_cmp(const void* a, const void* b) {
  const OrEntry* x = (const OrEntry*)a;
  const OrEntry* y = (const OrEntry*)b;
  const float mx = fabsf(x->v), my = fabsf(y->v);
  if (mx != my) return mx > my ? -1 : 1;
  return x->i < y->i ? -1 : (x->i > y->i ? 1 : 0);
}

/* topk_divide_conquer (sparsify.cpp:41-80): exact top-k under `precedes`, in that order.  The
   reference's chunked selection equals a full selection for every chunk count (its header,
   sparsify.hpp:22-28), so this restates it as one sort. */
int or_topk(uint64_t len, const float* t, uint64_t k, uint64_t* out_idx, float* out_val) {
  if (k > len) return OR_ERR_K_TOO_LARGE;
  if (k == 0) return OR_ERR_INVALID_ARGUMENT;
  OrEntry* e = (OrEntry*)malloc(len * sizeof(OrEntry));
  for (uint64_t i = 0; i < len; ++i) {
    e[i].v = t[i];
    e[i].i = i;
  }
  qsort(e, len, sizeof(OrEntry), or_precedes_cmp);
  for (uint64_t j = 0; j < k; ++j) {
    out_idx[j] = e[j].i;
    out_val[j] = e[j].v;
  }
  free(e);
  return OR_OK;
}

/* selected_count (sparsify.cpp:98-103) */
uint64_t or_selected_count(double ratio, uint64_t len) {
  if (len == 0) return 0;
  const double keep = (1.0 - ratio) * (double)len;
  uint64_t k = (uint64_t)ceil(keep);
  if (k < 1) k = 1;
  if (k > len) k = len;
  return k;
}

static int or_u64_cmp(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* CompressionState::compress_step (sparsify.cpp:120-161) on one layer's state, in place:
   velocity = momentum*velocity + grad; residual += velocity; emit the top selected_count
   residual entries in increasing index order; zero residual and velocity there. */
int or_dgc_step(uint64_t len, const float* g, float* vel, float* res, double ratio, float mom,
                uint64_t* out_idx, float* out_val, uint64_t* count) {
  if (len == 0) return OR_ERR_INVALID_ARGUMENT;
  for (uint64_t i = 0; i < len; ++i) {
    vel[i] = mom * vel[i] + g[i];
    res[i] += vel[i];
  }
  const uint64_t k = or_selected_count(ratio, len);
  uint64_t* idx = (uint64_t*)malloc(k * sizeof(uint64_t));
  float* val = (float*)malloc(k * sizeof(float));
  int rc = or_topk(len, res, k, idx, val);
  if (rc == OR_OK) {
    qsort(idx, k, sizeof(uint64_t), or_u64_cmp);
    for (uint64_t j = 0; j < k; ++j) {
      out_idx[j] = idx[j];
      out_val[j] = res[idx[j]];
    }
    for (uint64_t j = 0; j < k; ++j) {
      res[idx[j]] = 0.0f;
      vel[idx[j]] = 0.0f;
    }
    *count = k;
  }
  free(idx);
  free(val);
  return rc;
}
