// dgc.cu -- the paper's DGC gradient sparsification on device, beside the
// KNN-softmax path: topk_divide_conquer (sparsify.cpp:41-80) and the momentum-corrected
// CompressionState::compress_step (sparsify.cpp:120-161), bit-exact with the reference.
//
// Exact top-k under the reference's total order `precedes` (|value| descending, index
// ascending) does not depend on the chunking, so the device selects in one pass: every element
// becomes the 64-bit key (bits(|v|) << 32 | ~index) -- larger key = earlier in `precedes` --
// and a descending radix sort of the keys yields the selection order directly.
#include <cub/cub.cuh>

#include <cmath>
#include <string>
#include <unordered_map>
#include <vector>

#include "layer.cuh"

namespace xknn {
namespace {

__device__ __forceinline__ unsigned long long topk_key(float v, uint64_t i) {
  const uint32_t m = __float_as_uint(v) & 0x7fffffffu;  // |v|; -0 and +0 share a key
  return ((unsigned long long)m << 32) | (0xffffffffull - (uint32_t)i);
}

__global__ void k_topk_keys(const float* __restrict__ t, uint64_t len,
                            unsigned long long* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = topk_key(t[i], i);
}

// velocity <- momentum * velocity + grad; residual <- residual + velocity (sparsify.cpp:129-132,
// fp32, separate multiply and add); the residual's selection key
__global__ void k_dgc_accum(const float* __restrict__ g, float* __restrict__ vel,
                            float* __restrict__ res, uint64_t len, float mom,
                            unsigned long long* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float v = __fadd_rn(__fmul_rn(mom, vel[i]), g[i]);
    const float r = __fadd_rn(res[i], v);
    vel[i] = v;
    res[i] = r;
    keys[i] = topk_key(r, i);
  }
}

// the first k sorted keys -> (index, value) in selection order
__global__ void k_topk_take(const unsigned long long* __restrict__ sorted, uint64_t k,
                            const float* __restrict__ t, uint64_t* __restrict__ idx,
                            float* __restrict__ val, uint32_t* __restrict__ idx32) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < k;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = 0xffffffffu - (uint32_t)(sorted[j] & 0xffffffffull);
    if (idx) idx[j] = i;
    if (val) val[j] = t[i];
    if (idx32) idx32[j] = i;
  }
}

// ascending indices -> output pairs; factor masking of residual and velocity
// (sparsify.cpp:152-157)
__global__ void k_dgc_emit(const uint32_t* __restrict__ sorted_idx, uint64_t k,
                           float* __restrict__ res, float* __restrict__ vel,
                           uint64_t* __restrict__ out_idx, float* __restrict__ out_val) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < k;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = sorted_idx[j];
    out_idx[j] = i;
    out_val[j] = res[i];
  }
}
__global__ void k_dgc_mask(const uint32_t* __restrict__ sorted_idx, uint64_t k,
                           float* __restrict__ res, float* __restrict__ vel) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < k;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = sorted_idx[j];
    res[i] = 0.0f;
    vel[i] = 0.0f;
  }
}

struct Scratch {
  std::vector<void*> p;
  ~Scratch() {
    for (void* q : p) cudaFree(q);
  }
  template <typename T>
  cudaError_t get(T** out, uint64_t count) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<uint64_t>(count, 1) * sizeof(T));
    if (e == cudaSuccess) p.push_back(q);
    *out = static_cast<T*>(q);
    return e;
  }
};

#define D_CUDA(x)                                                                     \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) return fail_msg(XKNN_ERR_CUDA, cudaGetErrorString(e_));    \
  } while (0)

// sorts `keys` (len, device) descending into `sorted`
xknn_status_t sort_keys_desc(const unsigned long long* keys, unsigned long long* sorted,
                             uint64_t len, Scratch& mem, cudaStream_t s) {
  size_t tb = 0;
  void* tmp = nullptr;
  D_CUDA(cub::DeviceRadixSort::SortKeysDescending(nullptr, tb, keys, sorted, (int)len, 0, 64, s));
  D_CUDA(mem.get(reinterpret_cast<uint8_t**>(&tmp), tb));
  D_CUDA(cub::DeviceRadixSort::SortKeysDescending(tmp, tb, keys, sorted, (int)len, 0, 64, s));
  return XKNN_OK;
}

}  // namespace
}  // namespace xknn

// CompressionState: per-layer velocity and residual, device-resident
struct xknn_dgc {
  double ratio = 0.0;
  float momentum = 0.0f;
  cudaStream_t stream = nullptr;
  struct Buf {
    float* vel = nullptr;
    float* res = nullptr;
    uint64_t len = 0;
  };
  std::unordered_map<uint32_t, Buf> layers;
};

using xknn::fail_msg;

extern "C" {

uint64_t xknn_dgc_selected_count(double sparsity_ratio, uint64_t len) {
  // selected_count (sparsify.cpp:98-103), the same double arithmetic
  if (len == 0) return 0;
  const double keep = (1.0 - sparsity_ratio) * static_cast<double>(len);
  const uint64_t k = static_cast<uint64_t>(std::ceil(keep));
  return std::min<uint64_t>(std::max<uint64_t>(k, 1), len);
}

xknn_status_t xknn_topk(const float* values_dev, uint64_t len, uint64_t k, uint64_t* out_idx_dev,
                        float* out_val_dev, void* stream) {
  if (k > len) return fail_msg(XKNN_ERR_K_TOO_LARGE, "topk: k exceeds tensor length");
  if (k == 0) return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "topk: k must be positive");
  if (len >= 0xffffffffull || len > (uint64_t)INT32_MAX)
    return fail_msg(XKNN_ERR_UNSUPPORTED, "topk: tensor length must fit the 32-bit key index");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  xknn::Scratch mem;
  unsigned long long *keys = nullptr, *sorted = nullptr;
  D_CUDA(mem.get(&keys, len));
  D_CUDA(mem.get(&sorted, len));
  xknn::k_topk_keys<<<xknn::grid_for(len, 256), 256, 0, s>>>(values_dev, len, keys);
  D_CUDA(cudaGetLastError());
  xknn_status_t st = xknn::sort_keys_desc(keys, sorted, len, mem, s);
  if (st != XKNN_OK) return st;
  xknn::k_topk_take<<<xknn::grid_for(k, 256), 256, 0, s>>>(sorted, k, values_dev, out_idx_dev,
                                                           out_val_dev, nullptr);
  D_CUDA(cudaGetLastError());
  D_CUDA(cudaStreamSynchronize(s));
  return XKNN_OK;
}

xknn_status_t xknn_dgc_create(double sparsity_ratio, float momentum, void* stream,
                              xknn_dgc_t** out) {
  if (!out) return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "null output");
  if (sparsity_ratio < 0.0 || sparsity_ratio >= 1.0)
    return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "CompressionState: sparsity ratio must be in [0, 1)");
  auto* h = new xknn_dgc;
  h->ratio = sparsity_ratio;
  h->momentum = momentum;
  h->stream = static_cast<cudaStream_t>(stream);
  *out = h;
  return XKNN_OK;
}

xknn_status_t xknn_dgc_set_sparsity(xknn_dgc_t* h, double sparsity_ratio) {
  if (!h) return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "null handle");
  if (sparsity_ratio < 0.0 || sparsity_ratio >= 1.0)
    return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "CompressionState: sparsity ratio must be in [0, 1)");
  h->ratio = sparsity_ratio;
  return XKNN_OK;
}

xknn_status_t xknn_dgc_compress(xknn_dgc_t* h, uint32_t layer_id, const float* grad_dev,
                                uint64_t len, uint64_t* out_idx_dev, float* out_val_dev,
                                uint64_t* count) {
  if (!h) return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "null handle");
  if (len == 0) return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "compress_step: empty gradient");
  if (len > (uint64_t)INT32_MAX)
    return fail_msg(XKNN_ERR_UNSUPPORTED, "compress_step: layer length must fit 31 bits");
  cudaStream_t s = h->stream;
  auto it = h->layers.find(layer_id);
  if (it == h->layers.end()) {  // CompressionState::layer: zero state on first use
    xknn_dgc::Buf b;
    b.len = len;
    D_CUDA(cudaMalloc(&b.vel, len * sizeof(float)));
    D_CUDA(cudaMalloc(&b.res, len * sizeof(float)));
    D_CUDA(cudaMemsetAsync(b.vel, 0, len * sizeof(float), s));
    D_CUDA(cudaMemsetAsync(b.res, 0, len * sizeof(float), s));
    it = h->layers.emplace(layer_id, b).first;
  } else if (it->second.len != len) {
    return fail_msg(XKNN_ERR_SHAPE_MISMATCH,
                    ("compress_step: layer " + std::to_string(layer_id) + " length changed").c_str());
  }
  xknn_dgc::Buf& b = it->second;
  const uint64_t k = xknn_dgc_selected_count(h->ratio, len);
  xknn::Scratch mem;
  unsigned long long *keys = nullptr, *sorted = nullptr;
  uint32_t *sel = nullptr, *sel_sorted = nullptr;
  D_CUDA(mem.get(&keys, len));
  D_CUDA(mem.get(&sorted, len));
  D_CUDA(mem.get(&sel, k));
  D_CUDA(mem.get(&sel_sorted, k));
  xknn::k_dgc_accum<<<xknn::grid_for(len, 256), 256, 0, s>>>(grad_dev, b.vel, b.res, len,
                                                             h->momentum, keys);
  D_CUDA(cudaGetLastError());
  xknn_status_t st = xknn::sort_keys_desc(keys, sorted, len, mem, s);
  if (st != XKNN_OK) return st;
  xknn::k_topk_take<<<xknn::grid_for(k, 256), 256, 0, s>>>(sorted, k, b.res, nullptr, nullptr, sel);
  D_CUDA(cudaGetLastError());
  {  // the emitted entries in increasing index order (sparsify.cpp:143-151)
    size_t tb = 0;
    void* tmp = nullptr;
    D_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, sel, sel_sorted, (int)k, 0, 32, s));
    D_CUDA(mem.get(reinterpret_cast<uint8_t**>(&tmp), tb));
    D_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, sel, sel_sorted, (int)k, 0, 32, s));
  }
  xknn::k_dgc_emit<<<xknn::grid_for(k, 256), 256, 0, s>>>(sel_sorted, k, b.res, b.vel, out_idx_dev,
                                                          out_val_dev);
  xknn::k_dgc_mask<<<xknn::grid_for(k, 256), 256, 0, s>>>(sel_sorted, k, b.res, b.vel);
  D_CUDA(cudaGetLastError());
  D_CUDA(cudaStreamSynchronize(s));
  if (count) *count = k;
  return XKNN_OK;
}

xknn_status_t xknn_dgc_state(xknn_dgc_t* h, uint32_t layer_id, float* residual_dev,
                             float* velocity_dev, uint64_t len) {
  if (!h) return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "null handle");
  auto it = h->layers.find(layer_id);
  if (it == h->layers.end()) {  // residual(): zeros until first compressed
    if (residual_dev) D_CUDA(cudaMemsetAsync(residual_dev, 0, len * sizeof(float), h->stream));
    if (velocity_dev) D_CUDA(cudaMemsetAsync(velocity_dev, 0, len * sizeof(float), h->stream));
  } else {
    if (it->second.len != len) return fail_msg(XKNN_ERR_SHAPE_MISMATCH, "dgc_state: length");
    if (residual_dev)
      D_CUDA(cudaMemcpyAsync(residual_dev, it->second.res, len * 4, cudaMemcpyDeviceToDevice, h->stream));
    if (velocity_dev)
      D_CUDA(cudaMemcpyAsync(velocity_dev, it->second.vel, len * 4, cudaMemcpyDeviceToDevice, h->stream));
  }
  D_CUDA(cudaStreamSynchronize(h->stream));
  return XKNN_OK;
}

xknn_status_t xknn_dgc_destroy(xknn_dgc_t* h) {
  if (!h) return XKNN_OK;
  for (auto& kv : h->layers) {
    cudaFree(kv.second.vel);
    cudaFree(kv.second.res);
  }
  delete h;
  return XKNN_OK;
}

}  // extern "C"
