/* xknn_oracle.h -- C ABI of the CPU oracle (TEST INFRASTRUCTURE ONLY; see xknn_oracle.c). */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes share their numbering with include/xknn.h (errors.hpp classes). */
enum {
  OR_OK = 0,
  OR_ERR_SHAPE_MISMATCH = 1,
  OR_ERR_ZERO_NORM_ROW = 2,
  OR_ERR_LABEL_OUT_OF_RANGE = 3,
  OR_ERR_K_TOO_LARGE = 4,
  OR_ERR_EMPTY_SHARD = 5,
  OR_ERR_M_TOO_SMALL = 6,
  OR_ERR_LABEL_NOT_ACTIVE = 7,
  OR_ERR_INVALID_ARGUMENT = 8,
};

void or_shard_range(uint64_t n, uint64_t p, uint64_t s, uint64_t* begin, uint64_t* end);
uint64_t or_shard_of(uint64_t n, uint64_t p, uint64_t cls);
uint64_t or_compress_graph(uint64_t n, uint64_t k, const uint32_t* g_flat, uint64_t p,
                           uint64_t shard, uint32_t* k_per_class, uint64_t* offsets,
                           uint32_t* flat_out);
int or_select_active_full(uint64_t n, uint64_t k, const uint32_t* g_flat, const uint32_t* labels,
                          uint64_t b, uint64_t m_active, uint64_t seed, uint32_t* out,
                          uint64_t* out_count, int* contains_all);
int or_select_active_shards(uint64_t n, uint64_t p, const uint32_t* const* k_per_class,
                            const uint64_t* const* offsets, const uint32_t* const* flat,
                            const uint32_t* labels, uint64_t b, uint64_t m_active, uint64_t seed,
                            uint32_t* out, uint64_t* out_count, int* contains_all);
int or_select_active_shards_stream(uint64_t n, uint64_t p, const uint32_t* const* k_per_class,
                                   const uint64_t* const* offsets, const uint32_t* const* flat,
                                   const uint32_t* labels, uint64_t b, uint64_t m_active,
                                   const uint64_t* words, uint64_t nwords, uint32_t* out,
                                   uint64_t* out_count, int* contains_all);
int or_l2_normalize_rows(uint64_t rows, uint64_t cols, const float* in, float eps, float* out,
                         float* norms, uint64_t* bad_row);
void or_l2_normalize_backward(uint64_t rows, uint64_t cols, const float* nrm, const float* norms,
                              const float* g_in, float* g_out);
void or_matmul_nt(uint64_t m, uint64_t n, uint64_t kd, const float* a, const float* b, float* c);
void or_matmul_nn(uint64_t m, uint64_t n, uint64_t kd, const float* a, const float* b, float* c);
void or_matmul_tn(uint64_t rows, uint64_t ac, uint64_t bc, const float* a, const float* b,
                  float* c);
int or_softmax_xent(uint64_t m, uint64_t c, const float* logits, const uint32_t* labels,
                    double* loss, float* grad);
int or_knn_softmax_forward_backward(uint64_t b, uint64_t n, uint64_t d, const float* x,
                                    const float* w, const uint32_t* labels, const uint32_t* active,
                                    uint64_t m_act, float scale, double* loss, float* grad_logits,
                                    float* grad_features, float* grad_w_active);
int or_distributed_softmax_xent_cols(uint64_t p, uint64_t m, const float* const* logits,
                                     const uint32_t* const* cols, const uint64_t* ncols,
                                     const uint32_t* labels, double* loss, float* const* grads);
void or_sgd_step_rows(uint64_t cols, float* params, const float* grad_rows, float* velocity,
                      const uint32_t* rows, uint64_t nrows, float lr, float momentum, float wd);
int or_build_graph_bruteforce(uint64_t n, uint64_t d, const float* w, uint64_t k, uint32_t* out);
int or_classify_retrieval(uint64_t nq, uint64_t n, uint64_t d, const float* q, const float* w,
                          uint32_t* out_class, float* out_score);
int or_topk(uint64_t len, const float* t, uint64_t k, uint64_t* out_idx, float* out_val);
uint64_t or_selected_count(double ratio, uint64_t len);
int or_dgc_step(uint64_t len, const float* g, float* vel, float* res, double ratio, float mom,
                uint64_t* out_idx, float* out_val, uint64_t* count);
void or_graph_rows_update(uint64_t nq, uint64_t d, const float* q, const uint64_t* qid, uint64_t k,
                          const float* chunk, uint64_t rows, uint64_t base, float* sc, uint32_t* ix,
                          uint64_t* sz);
int or_graph_row(uint64_t n, uint64_t d, const float* w, uint64_t j, uint64_t k, uint32_t* out);
int or_fc_train_step(uint64_t n, uint64_t d, uint64_t p, float* w, float* velocity,
                     const float* x, const uint32_t* labels, uint64_t b,
                     const uint32_t* const* k_per_class, const uint64_t* const* offsets,
                     const uint32_t* const* flat, uint64_t m_active, uint64_t seed, float scale,
                     float lr, float momentum, float wd, double* loss_out, uint32_t* active_out,
                     uint64_t* active_count, float* grad_feat, float* logits_out);
int or_fc_train_step_mb(uint64_t n, uint64_t d, uint64_t p, float* w, float* velocity,
                        const float* x, const uint32_t* labels, uint64_t b,
                        const uint32_t* const* k_per_class, const uint64_t* const* offsets,
                        const uint32_t* const* flat, uint64_t m_active, uint64_t seed,
                        float scale, float lr, float momentum, float wd, uint64_t micro_batches,
                        double* loss_out, uint32_t* active_out, uint64_t* active_count,
                        float* grad_feat);
/* raw mt19937_64 / uniform_int stream, for testing the device generator */
void or_mt64_stream(uint64_t seed, uint64_t count, uint64_t* out);
void or_uniform_picks(uint64_t seed, uint64_t csize, uint64_t need, uint64_t* out);

#ifdef __cplusplus
}
#endif
