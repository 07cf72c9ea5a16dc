// exact.cu -- XKNN_PREC_FP32_EXACT: the three fc GEMMs on CUDA cores in the reference's
// summation order, and the distributed softmax-CE statistics (both precisions).
//
//   logits  = matmul(f_hat, w_sub, transpose_b) * s     matrix.cpp:57-68, parallel.cpp:550-551
//   dW_sub  = matmul_at(G, f_hat) * (s*weight)          matrix.cpp:84-98, parallel.cpp:564-566
//   dX_part = matmul(G, w_sub) * s                      matrix.cpp:69-80, parallel.cpp:568-569
//   softmax = distributed_softmax_xent_cols             parallel.cpp:106-188
//
// Each output element is accumulated sequentially over the inner index with separately rounded
// multiply and add (__fmul_rn/__fadd_rn, no FMA), so logits are bit-identical to the
// reference's; the softmax uses CUDA expf (<= 2 ulp from glibc), hence the 1e-5 tolerance.
#include "kernels.cuh"

namespace xknn {

namespace {

constexpr int kT = 16;   // output tile edge
constexpr int kKc = 32;  // inner chunk

// C[i][j] = (sum_k A[i][k] * B[j][k]) * scale   (A: rows x d, B: cols x d)
__global__ void k_gemm_nt_exact(const float* __restrict__ A, const float* __restrict__ Bm,
                                uint64_t rows, const unsigned int* cols_dev, uint32_t d,
                                float scale, float* __restrict__ C) {
  griddep_wait();
  const uint64_t cols = *cols_dev;
  __shared__ float As[kT][kKc + 1];
  __shared__ float Bs[kT][kKc + 1];
  const uint32_t tx = threadIdx.x, ty = threadIdx.y;
  const uint64_t ntile_j = (cols + kT - 1) / kT;
  const uint64_t ntiles = ((rows + kT - 1) / kT) * ntile_j;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t i0 = (tile / ntile_j) * kT, j0 = (tile % ntile_j) * kT;
    float acc = 0.0f;
    for (uint32_t k0 = 0; k0 < d; k0 += kKc) {
      for (uint32_t e = ty * kT + tx; e < kT * kKc; e += kT * kT) {
        const uint32_t r = e / kKc, c = e % kKc;
        As[r][c] = (i0 + r < rows) ? A[(i0 + r) * d + k0 + c] : 0.0f;
        Bs[r][c] = (j0 + r < cols) ? Bm[(j0 + r) * d + k0 + c] : 0.0f;
      }
      __syncthreads();
#pragma unroll 8
      for (int k = 0; k < kKc; ++k) acc = __fadd_rn(acc, __fmul_rn(As[ty][k], Bs[tx][k]));
      __syncthreads();
    }
    const uint64_t i = i0 + ty, j = j0 + tx;
    if (i < rows && j < cols) C[i * cols + j] = __fmul_rn(acc, scale);
  }
}

// dW[j][l] = ((sum_i G[i][j] * X[i][l]) * sw) ; G is rows x cols (row stride cols)
__global__ void k_gemm_tn_exact(const float* __restrict__ G, const float* __restrict__ X,
                                uint64_t rows, const unsigned int* cols_dev, uint32_t d, float sw,
                                float* __restrict__ out) {
  griddep_wait();
  const uint64_t cols = *cols_dev;
  const uint64_t total = cols * d;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = e / d, l = e % d;
    float acc = 0.0f;
    for (uint64_t i = 0; i < rows; ++i) acc = __fadd_rn(acc, __fmul_rn(G[i * cols + j], X[i * d + l]));
    // gw *= scale*weight, then axpy into the zeroed fc_acc (0 + 1*gw)
    out[e] = __fadd_rn(0.0f, __fmul_rn(1.0f, __fmul_rn(acc, sw)));
  }
}

// dX[i][l] = (sum_j G[i][j] * Wsub[j][l]) * s
__global__ void k_gemm_nn_exact(const float* __restrict__ G, const float* __restrict__ Wsub,
                                uint64_t rows, const unsigned int* cols_dev, uint32_t d,
                                float scale, float* __restrict__ out) {
  griddep_wait();
  const uint64_t cols = *cols_dev;
  const uint64_t total = rows * d;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = e / d, l = e % d;
    float acc = 0.0f;
    for (uint64_t j = 0; j < cols; ++j)
      acc = __fadd_rn(acc, __fmul_rn(G[i * cols + j], Wsub[j * d + l]));
    out[e] = __fmul_rn(acc, scale);
  }
}

// ---- distributed softmax statistics (parallel.cpp:123-156): one warp per row
__global__ void k_rowmax(const float* __restrict__ L, uint64_t rows, const unsigned int* cols_dev,
                         float* __restrict__ rowmax) {
  griddep_wait();
  griddep_launch();
  const uint64_t cols = *cols_dev;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < rows;
       i += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    float mx = -INFINITY;
    for (uint64_t j = lane; j < cols; j += 32) mx = fmaxf(mx, L[i * cols + j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(XKNN_FULL_MASK, mx, o));
    if (lane == 0) rowmax[i] = mx;
  }
}

// red[i] = sum_j double(expf(l - mx)), red[B+i] = double(l_y - mx), red[2B+i] = owner
__global__ void k_rowsum(const float* __restrict__ L, uint64_t rows, const unsigned int* cols_dev,
                         const float* __restrict__ rowmax, const int32_t* __restrict__ label_col,
                         double* __restrict__ red) {
  griddep_wait();
  griddep_launch();
  const uint64_t cols = *cols_dev;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < rows;
       i += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const float mx = rowmax[i];
    double s = 0.0;
    for (uint64_t j = lane; j < cols; j += 32) s += (double)expf(__fsub_rn(L[i * cols + j], mx));
    s = warp_sum(s);
    if (lane == 0) {
      red[i] = s;
      const int32_t c = label_col[i];
      red[rows + i] = c >= 0 ? (double)__fsub_rn(L[i * cols + c], mx) : 0.0;
      red[2 * rows + i] = c >= 0 ? 1.0 : 0.0;
    }
  }
}

// loss = mean_i(log(denom_i) - term_i) in row order (parallel.cpp:157-166); owner count must be
// exactly one per row.
__global__ void k_loss(const double* __restrict__ red, uint64_t rows, double* loss,
                       SelState* st, unsigned long long* err) {
  griddep_wait();
  griddep_launch();
  __shared__ double part[256];
  double s = 0.0;
  // fixed-order blocked sum: thread t sums rows [t*c, (t+1)*c) sequentially
  const uint64_t chunk = (rows + blockDim.x - 1) / blockDim.x;
  for (uint64_t i = threadIdx.x * chunk; i < min(rows, (threadIdx.x + 1) * chunk); ++i) {
    if (red[2 * rows + i] != 1.0) raise_error(err, XKNN_ERR_LABEL_OUT_OF_RANGE, i);
    s += log(red[i]) - red[rows + i];
  }
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (uint32_t k = 0; k < blockDim.x; ++k) t += part[k];
    const double l = t / (double)rows;
    *loss = l;
    st->loss = l;
  }
}

// G = expf(l - mx) * float(1/denom) * (1/m); label column -= 1/m   (parallel.cpp:168-186)
__global__ void k_softmax_grad(float* __restrict__ L, uint64_t rows, const unsigned int* cols_dev,
                               const float* __restrict__ rowmax, const double* __restrict__ red,
                               const int32_t* __restrict__ label_col) {
  griddep_wait();
  const uint64_t cols = *cols_dev;
  const float inv_m = 1.0f / (float)rows;
  const uint64_t total = rows * cols;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = e / cols, j = e % cols;
    const float inv_denom = (float)(1.0 / red[i]);
    float g = __fmul_rn(__fmul_rn(expf(__fsub_rn(L[e], rowmax[i])), inv_denom), inv_m);
    if (label_col[i] == (int32_t)j) g = __fsub_rn(g, inv_m);
    L[e] = g;
  }
}

}  // namespace

cudaError_t launch_logits_exact(const float* xhat, const float* wsub, uint64_t rows,
                                const unsigned int* cols, uint64_t max_cols, uint32_t d,
                                float scale, float* out, cudaStream_t s) {
  const uint64_t tiles = ((rows + kT - 1) / kT) * ((max_cols + kT - 1) / kT);
  launch_pdl(k_gemm_nt_exact, grid_for(tiles, 1, 148u * 64u), dim3(kT, kT), 0, s, xhat, wsub, rows, cols,
                                                                           d, scale, out);
  return cudaGetLastError();
}

cudaError_t launch_dw_exact(const float* G, const float* xhat, uint64_t rows,
                            const unsigned int* cols, uint64_t max_cols, uint32_t d, float sw,
                            float* out, cudaStream_t s) {
  launch_pdl(k_gemm_tn_exact, grid_for(max_cols * d, 256, 148u * 64u), 256, 0, s, G, xhat, rows, cols, d,
                                                                          sw, out);
  return cudaGetLastError();
}

cudaError_t launch_dx_exact(const float* G, const float* wsub, uint64_t rows,
                            const unsigned int* cols, uint32_t d, float scale, float* out,
                            cudaStream_t s) {
  launch_pdl(k_gemm_nn_exact, grid_for(rows * d, 256, 148u * 64u), 256, 0, s, G, wsub, rows, cols, d,
                                                                      scale, out);
  return cudaGetLastError();
}

cudaError_t launch_rowmax(const float* L, uint64_t rows, const unsigned int* cols, float* rowmax,
                          cudaStream_t s) {
  launch_pdl(k_rowmax, grid_for(rows * 32, 256), 256, 0, s, L, rows, cols, rowmax);
  return cudaGetLastError();
}

cudaError_t launch_rowsum(const float* L, uint64_t rows, const unsigned int* cols,
                          const float* rowmax, const int32_t* label_col, double* red,
                          cudaStream_t s) {
  launch_pdl(k_rowsum, grid_for(rows * 32, 256), 256, 0, s, L, rows, cols, rowmax, label_col, red);
  return cudaGetLastError();
}

cudaError_t launch_loss(const double* red, uint64_t rows, double* loss, SelState* st,
                        unsigned long long* err, cudaStream_t s) {
  launch_pdl(k_loss, 1, 256, 0, s, red, rows, loss, st, err);
  return cudaGetLastError();
}

cudaError_t launch_softmax_grad(float* L, uint64_t rows, const unsigned int* cols,
                                uint64_t max_cols, const float* rowmax, const double* red,
                                const int32_t* label_col, cudaStream_t s) {
  launch_pdl(k_softmax_grad, grid_for(rows * max_cols, 256), 256, 0, s, L, rows, cols, rowmax, red,
                                                                label_col);
  return cudaGetLastError();
}

}  // namespace xknn
