// standalone.cu -- the reference's single-device free functions of the hot path, outside the
// sharded layer object:
//
//   xknn_select_full_graph      select_active_classes(const KnnGraph&, ...)
//                               (knn_softmax.cpp:100-115 + finish_selection :17-81): ranks are
//                               positions in the FULL neighbour lists; equal to the shard overload
//                               only at P = 1 (knn_softmax.hpp:40-43).  Runs the layer's device
//                               selection (select.cu) on a select-only P = 1 layer whose graph is
//                               the uncompressed N x k list.
//   xknn_knn_softmax_fwd_bwd    knn_softmax_forward_backward (knn_softmax.cpp:136-186): gather of
//                               the active rows of w_norm, logits = matmul(x_norm, w_active, T) *
//                               scale, softmax_xent (softmax.cpp:8-39), grad_features =
//                               matmul(G, w_active) * scale, grad_weights = matmul_at(G, x_norm) *
//                               scale on the active rows.  fp32 on CUDA cores in the reference's
//                               summation order (exact.cu): logits bit-identical.
#include <string>
#include <vector>

#include "kernels.cuh"

namespace xknn {
namespace {

// w_active[i] = w_norm[active[i]] (knn_softmax.cpp:147-153); LabelOutOfRange for an active class
// outside [0, n)
__global__ void k_gather_active(const float* __restrict__ w, uint64_t n, uint32_t d,
                                const uint32_t* __restrict__ active, uint64_t m,
                                float* __restrict__ out, unsigned long long* err) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < m;
       i += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint32_t c = active[i];
    if (c >= n) {
      if (lane == 0) raise_error(err, XKNN_ERR_LABEL_OUT_OF_RANGE, i);
      continue;
    }
    for (uint32_t j = lane; j < d; j += 32) out[i * d + j] = w[(uint64_t)c * d + j];
  }
}

// ActiveSet::position_of (knn_softmax.cpp:85-90) of every label; LabelNotActive if missing
__global__ void k_label_positions(const uint32_t* __restrict__ labels, uint64_t b,
                                  const uint32_t* __restrict__ active, uint64_t m,
                                  int32_t* __restrict__ col, unsigned long long* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < b;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t y = labels[i];
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (active[mid] < y) lo = mid + 1; else hi = mid;
    }
    if (lo < m && active[lo] == y) {
      col[i] = (int32_t)lo;
    } else {
      col[i] = -1;
      raise_error(err, XKNN_ERR_LABEL_NOT_ACTIVE, i);
    }
  }
}

struct DevScratch {
  cudaStream_t s;
  std::vector<void*> ptrs;
  template <typename T>
  cudaError_t get(T** p, uint64_t count) {
    void* v = nullptr;
    cudaError_t e = cudaMallocAsync(&v, (count ? count : 1) * sizeof(T), s);
    if (e == cudaSuccess) ptrs.push_back(v);
    *p = static_cast<T*>(v);
    return e;
  }
  ~DevScratch() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

xknn_status_t cuda_status(cudaError_t e, const char* what) {
  (void)cudaGetLastError();
  return fail_msg(e == cudaErrorMemoryAllocation ? XKNN_ERR_OUT_OF_MEMORY : XKNN_ERR_CUDA,
                  (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
}

}  // namespace
}  // namespace xknn

#define SA_CUDA(expr)                                         \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return xknn::cuda_status(_e, #expr); \
  } while (0)

extern "C" {

xknn_status_t xknn_select_full_graph(const uint32_t* graph_dev, uint64_t num_classes, uint32_t k,
                                     const uint32_t* labels_dev, uint64_t batch,
                                     uint64_t m_active, uint64_t seed, uint32_t* out_active_dev,
                                     uint64_t* count_host, int* contains_all_host,
                                     void* stream) {
  if (num_classes == 0 || batch == 0)
    return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "select_active_classes: empty graph or batch");
  if (m_active > num_classes)
    return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "select_active_classes: M exceeds the class count");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  xknn_config_t cfg{};
  cfg.scale = 1.f;
  cfg.m_active = m_active;
  cfg.rng_seed = seed;
  cfg.max_batch = batch;
  cfg.precision = XKNN_PREC_FP32_EXACT;
  cfg.flags = XKNN_FLAG_SELECT_ONLY | XKNN_FLAG_NO_GRAPH;
  xknn_layer_t* h = nullptr;
  xknn_status_t st = xknn_layer_create(0, 1, num_classes, 128, &cfg, nullptr, stream, &h);
  if (st != XKNN_OK) return st;
  // the uncompressed graph as a one-shard CSR: k entries per class, positions = full-list ranks
  uint32_t* kpc = nullptr;
  uint64_t* off = nullptr;
  cudaError_t e = cudaMallocAsync(&kpc, num_classes * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&off, num_classes * 8, s);
  if (e == cudaSuccess) {
    std::vector<uint32_t> hk(num_classes, k);
    std::vector<uint64_t> ho(num_classes);
    for (uint64_t c = 0; c < num_classes; ++c) ho[c] = c * (uint64_t)k;
    e = cudaMemcpyAsync(kpc, hk.data(), num_classes * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(off, ho.data(), num_classes * 8, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  if (e != cudaSuccess) st = xknn::cuda_status(e, "select_full_graph scratch");
  if (st == XKNN_OK)
    st = xknn_layer_set_graph_csr(h, kpc, off, graph_dev, num_classes * (uint64_t)k, 1);
  if (st == XKNN_OK)
    st = xknn_select(h, labels_dev, batch, out_active_dev, count_host, contains_all_host);
  if (kpc) cudaFreeAsync(kpc, s);
  if (off) cudaFreeAsync(off, s);
  xknn_layer_destroy(h);
  return st;
}

xknn_status_t xknn_knn_softmax_fwd_bwd(const float* x_norm_dev, uint64_t batch,
                                       const float* w_norm_dev, uint64_t num_classes,
                                       uint64_t dim, const uint32_t* labels_dev,
                                       const uint32_t* active_dev, uint64_t m_act, float scale,
                                       double* loss_host, float* grad_logits_dev,
                                       float* grad_features_dev, float* grad_w_active_dev,
                                       void* stream) {
  using namespace xknn;
  if (dim == 0 || dim % 128 != 0 || dim > 1024)
    return fail_msg(XKNN_ERR_SHAPE_MISMATCH, "knn_softmax: dim must be a multiple of 128, <= 1024");
  if (batch == 0) return fail_msg(XKNN_ERR_SHAPE_MISMATCH, "knn_softmax: one label per row required");
  if (m_act == 0) return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "knn_softmax: empty active set");
  if (m_act >= (1ull << 31)) return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "knn_softmax: active set too large");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t d = (uint32_t)dim;
  DevScratch mem{s, {}};
  float *wsub, *L, *rowmax, *gx;
  double *red, *loss;
  int32_t* col;
  unsigned int* cols;
  unsigned long long* err;
  SelState* st;
  SA_CUDA(mem.get(&wsub, m_act * d));
  SA_CUDA(mem.get(&L, batch * m_act));
  SA_CUDA(mem.get(&rowmax, batch));
  SA_CUDA(mem.get(&red, 3 * batch));
  SA_CUDA(mem.get(&loss, 1));
  SA_CUDA(mem.get(&col, batch));
  SA_CUDA(mem.get(&cols, 1));
  SA_CUDA(mem.get(&err, 1));
  SA_CUDA(mem.get(&st, 1));
  SA_CUDA(mem.get(&gx, grad_logits_dev ? 1 : batch * m_act));
  float* G = grad_logits_dev ? grad_logits_dev : gx;
  const unsigned int mc = (unsigned int)m_act;
  SA_CUDA(cudaMemcpyAsync(cols, &mc, 4, cudaMemcpyHostToDevice, s));
  SA_CUDA(cudaMemsetAsync(err, 0, 8, s));
  k_gather_active<<<grid_for(m_act * 32, 256), 256, 0, s>>>(w_norm_dev, num_classes, d, active_dev,
                                                            m_act, wsub, err);
  SA_CUDA(cudaGetLastError());
  k_label_positions<<<grid_for(batch, 256), 256, 0, s>>>(labels_dev, batch, active_dev, m_act, col,
                                                         err);
  SA_CUDA(cudaGetLastError());
  unsigned long long w = 0;
  SA_CUDA(cudaMemcpyAsync(&w, err, 8, cudaMemcpyDeviceToHost, s));
  SA_CUDA(cudaStreamSynchronize(s));
  if (w)  // the reference throws before any arithmetic
    return fail_row((xknn_status_t)(w & 0xff),
                    (w & 0xff) == XKNN_ERR_LABEL_NOT_ACTIVE
                        ? "knn_softmax: label missing from the active set"
                        : "knn_softmax: active class out of range",
                    w >> 8);
  // logits = matmul(x_norm, w_active, T) * scale; softmax_xent; both gradients
  SA_CUDA(launch_logits_exact(x_norm_dev, wsub, batch, cols, m_act, d, scale, L, s));
  SA_CUDA(launch_rowmax(L, batch, cols, rowmax, s));
  SA_CUDA(launch_rowsum(L, batch, cols, rowmax, col, red, s));
  SA_CUDA(launch_loss(red, batch, loss, st, err, s));
  SA_CUDA(cudaMemcpyAsync(G, L, batch * m_act * 4, cudaMemcpyDeviceToDevice, s));
  SA_CUDA(launch_softmax_grad(G, batch, cols, m_act, rowmax, red, col, s));
  SA_CUDA(launch_dx_exact(G, wsub, batch, cols, d, scale, grad_features_dev, s));
  SA_CUDA(launch_dw_exact(G, x_norm_dev, batch, cols, m_act, d, scale, grad_w_active_dev, s));
  double lh = 0;
  SA_CUDA(cudaMemcpyAsync(&lh, loss, 8, cudaMemcpyDeviceToHost, s));
  SA_CUDA(cudaMemcpyAsync(&w, err, 8, cudaMemcpyDeviceToHost, s));
  SA_CUDA(cudaStreamSynchronize(s));
  if (w) return fail_msg((xknn_status_t)(w & 0xff), "knn_softmax: device error");
  if (loss_host) *loss_host = lh;
  return XKNN_OK;
}

}  // extern "C"
