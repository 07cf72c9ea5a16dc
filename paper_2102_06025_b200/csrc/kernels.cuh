// kernels.cuh -- host launchers of the device kernels (all asynchronous on `s`).
#pragma once
#include "layer.cuh"

namespace xknn {

// rowops.cu
// The one-hot part of the softmax gradient on the weight side (tensor-core precisions): for
// active column t, dW[t] -= sb * sum{x_hat_b : b in the list head[t] -> next[b] -> ...}, summed
// in ascending b; the update clears head[t] (-1) for the next step.  head == nullptr: none.
struct LabelFix {
  int32_t* head = nullptr;
  const int32_t* next = nullptr;
  const float* X = nullptr;      // gathered raw features (B x D)
  const float* xnorm = nullptr;  // their norms
  float sb = 0.f;                // s / B
  // GEMM-dW tail split (dw_split): the rows of the last, partial wave of 256-class units arrive
  // as dw_split().s fp32 K-partials [slot][256][D] instead of dW rows; nullptr: none
  const float* dw_part = nullptr;
  uint32_t npairs = 0;
};

// GEMM-dW units are 256 active classes with the whole batch as K; their count rarely fills the
// 74 CTA pairs in whole waves (C2: 391 units = 5.28 waves).  The `tail` units of the last wave
// are split along K into s parts (s * tail <= npairs, s <= 4), each writing an fp32 partial that
// the row update sums in part order; `full` units run whole.
struct DwSplit {
  uint32_t full, s;
};
__host__ __device__ __forceinline__ DwSplit dw_split(uint32_t units, uint32_t npairs) {
  const uint32_t tail = units % npairs;
  uint32_t s = tail ? npairs / tail : 1;
  s = s > 4 ? 4 : (s < 1 ? 1 : s);
  if (s == 1) return {units, 1};
  return {units - tail, s};
}
cudaError_t launch_normalize_rows(const float* in, uint64_t rows, uint32_t d,
                                  const uint32_t* row_ids, const unsigned int* count,
                                  uint64_t id_base, float* out32, __nv_bfloat16* out16,
                                  float* norms, unsigned long long* err, cudaStream_t s,
                                  bool seq = false, float* out_lo = nullptr,
                                  __nv_bfloat16* out16_lo = nullptr, __nv_bfloat16* out_d = nullptr);
cudaError_t launch_update_rows(float* W, float* V, const float* G, const uint32_t* active,
                               const unsigned int* count, uint64_t max_rows, uint64_t begin,
                               uint32_t d, const float* wnorm, const float* lr, float mu, float wd,
                               const unsigned long long* err, cudaStream_t s,
                               unsigned max_grid = 148u * 16u, LabelFix lf = {});
cudaError_t launch_update_rows_bf16(float* W, float* V, const __nv_bfloat16* G,
                                    const uint32_t* active, const unsigned int* count,
                                    uint64_t max_rows, uint64_t begin, uint32_t d,
                                    const float* wnorm, const float* lr, float mu, float wd,
                                    const unsigned long long* err, cudaStream_t s,
                                    LabelFix lf = {});
cudaError_t launch_feature_backward(const float* X, const float* xnorm, const float* G,
                                    uint64_t rows, uint32_t d, float* out, cudaStream_t s,
                                    uint32_t micros = 1);

// exact.cu
cudaError_t launch_logits_exact(const float* xhat, const float* wsub, uint64_t rows,
                                const unsigned int* cols, uint64_t max_cols, uint32_t d,
                                float scale, float* out, cudaStream_t s);
cudaError_t launch_dw_exact(const float* G, const float* xhat, uint64_t rows,
                            const unsigned int* cols, uint64_t max_cols, uint32_t d, float sw,
                            float* out, cudaStream_t s);
cudaError_t launch_dx_exact(const float* G, const float* wsub, uint64_t rows,
                            const unsigned int* cols, uint32_t d, float scale, float* out,
                            cudaStream_t s);
cudaError_t launch_rowmax(const float* L, uint64_t rows, const unsigned int* cols, float* rowmax,
                          cudaStream_t s);
cudaError_t launch_rowsum(const float* L, uint64_t rows, const unsigned int* cols,
                          const float* rowmax, const int32_t* label_col, double* red,
                          cudaStream_t s);
cudaError_t launch_loss(const double* red, uint64_t rows, double* loss, SelState* st,
                        unsigned long long* err, cudaStream_t s);
cudaError_t launch_softmax_grad(float* L, uint64_t rows, const unsigned int* cols,
                                uint64_t max_cols, const float* rowmax, const double* red,
                                const int32_t* label_col, cudaStream_t s);

}  // namespace xknn

namespace xknn {
// fast.cu: pieces shared by the BF16 and FP32 (3xTF32) tensor-core paths
cudaError_t launch_rowreduce(const SelState* st, const float* partial, const float* labelterm,
                             const int32_t* lcol, uint32_t B, uint32_t bpad, double* red,
                             cudaStream_t s);
cudaError_t launch_dx_reduce(const float* partial, const double* red, uint32_t B, uint32_t nbt,
                             uint32_t splits, float scale, const int32_t* lcol,
                             const uint32_t* active, uint64_t begin, const float* W,
                             const float* wnorm, float* out, cudaStream_t s);
uint32_t gemm_pair_splits(uint32_t nbp, uint32_t max_units, uint32_t streams = 74);
}  // namespace xknn
