// graph.cu -- exact KNN class graph on device: build_graph_bruteforce (knn_graph.cpp:124-145)
// with the reference's ordering `better` (:20-26): self first, then descending inner product,
// ties to the lower class index.  Bit-exact with the reference:
//   1. candidates: bf16 CTA-pair GEMM of the normalized weights against themselves with a
//      threshold top-k' epilogue (fast.cu, k_gemm2<kG>): every column left out of a row's
//      candidate set has approximate score <= T_row;
//   2. exact re-score of the candidates in the reference's arithmetic (fp32, ascending d,
//      separate multiply and add), sort under `better`, keep k;
//   3. certificate: if the k-th exact score exceeds T_row + eps (eps bounds |bf16 GEMM - fp32
//      reference|, 2^-8 for unit rows plus accumulation terms), no left-out column can belong
//      to the top k; otherwise the row is recomputed by an exact scan over all N columns.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"

namespace xknn {

cudaError_t launch_graph_candidates(const __nv_bfloat16* Wb, uint32_t n, uint32_t npad,
                                    float2* cand, uint32_t* cnt, float* tau, uint32_t ch,
                                    uint32_t kprime, cudaStream_t s);

namespace {

constexpr float kEps = 0.0041f;  // >= 2^-8 (bf16 inputs, unit rows) + 2 * 512 * 2^-24

__global__ void k_to_bf16(const float* __restrict__ w, uint64_t n, uint64_t npad, uint32_t d,
                          __nv_bfloat16* __restrict__ out) {
  const uint64_t total = npad * d / 2;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = (2 * e) / d;
    float2 v = row < n ? reinterpret_cast<const float2*>(w)[e] : make_float2(0.f, 0.f);
    reinterpret_cast<__nv_bfloat162*>(out)[e] = __floats2bfloat162_rn(v.x, v.y);
  }
}

// the reference's score: dot += wj[d] * wi[d], d ascending, fp32 (knn_graph.cpp:137-138)
__device__ __forceinline__ float exact_dot(const float* __restrict__ a, const float* __restrict__ b,
                                           uint32_t d) {
  float acc = 0.0f;
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll 4
  for (uint32_t t = 0; t < d / 4; ++t) {
    const float4 x = a4[t], y = b4[t];
    acc = __fadd_rn(acc, __fmul_rn(x.x, y.x));
    acc = __fadd_rn(acc, __fmul_rn(x.y, y.y));
    acc = __fadd_rn(acc, __fmul_rn(x.z, y.z));
    acc = __fadd_rn(acc, __fmul_rn(x.w, y.w));
  }
  return acc;
}

// `better` without self (self is placed first separately): higher score, then lower index
__device__ __forceinline__ bool before(float sa, uint32_t ia, float sb, uint32_t ib) {
  if (sa != sb) return sa > sb;
  return ia < ib;
}

// One warp per row: exact re-score of its <= 2*ch candidates, warp bitonic sort, top k,
// certificate.  Shared memory per warp: 2*ch (score, index) pairs, padded to a power of two.
__global__ void k_graph_finalize(const float* __restrict__ wn, uint32_t n, uint32_t d,
                                 const float2* __restrict__ cand, const uint32_t* __restrict__ cnt,
                                 const float* __restrict__ tau, uint32_t ch, uint32_t k,
                                 uint32_t* __restrict__ out, uint32_t* fail_count,
                                 uint32_t* __restrict__ fail_list) {
  extern __shared__ uint8_t sm[];
  const uint32_t warps = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t cap = 1;
  while (cap < 2 * ch) cap <<= 1;
  float* ss = reinterpret_cast<float*>(sm) + (uint64_t)w * cap;
  uint32_t* si = reinterpret_cast<uint32_t*>(reinterpret_cast<float*>(sm) + (uint64_t)warps * cap) +
                 (uint64_t)w * cap;
  for (uint32_t j = blockIdx.x * warps + w; j < n; j += gridDim.x * warps) {
    const uint32_t c0 = cnt[2 * j], c1 = cnt[2 * j + 1];
    const uint32_t m = c0 + c1;
    const float T = fmaxf(tau[2 * j], tau[2 * j + 1]);
    const float* wj = wn + (uint64_t)j * d;
    for (uint32_t e = lane; e < cap; e += 32) {
      if (e < m) {
        const float2 c = e < c0 ? cand[(uint64_t)j * 2 * ch + e]
                                : cand[((uint64_t)j * 2 + 1) * ch + (e - c0)];
        const uint32_t i = __float_as_uint(c.y);
        ss[e] = exact_dot(wj, wn + (uint64_t)i * d, d);
        si[e] = i;
      } else {
        ss[e] = -INFINITY;
        si[e] = 0xffffffffu;
      }
    }
    __syncwarp();
    // bitonic sort, descending under `before`
    for (uint32_t size = 2; size <= cap; size <<= 1) {
      for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (uint32_t e = lane; e < cap; e += 32) {
          const uint32_t p = e ^ stride;
          if (p > e) {
            const bool dir = (e & size) == 0;  // true: this pair sorts "before" first
            const bool swp = dir ? before(ss[p], si[p], ss[e], si[e])
                                 : before(ss[e], si[e], ss[p], si[p]);
            if (swp) {
              const float ts = ss[e];
              ss[e] = ss[p];
              ss[p] = ts;
              const uint32_t ti = si[e];
              si[e] = si[p];
              si[p] = ti;
            }
          }
        }
        __syncwarp();
      }
    }
    // self first, then the k-1 best candidates
    bool ok = true;
    if (k > 1) ok = m >= k - 1 && ss[k - 2] > T + kEps;
    if (ok) {
      uint32_t* o = out + (uint64_t)j * k;
      for (uint32_t e = lane; e < k; e += 32) o[e] = e == 0 ? j : si[e - 1];
    } else if (lane == 0) {
      fail_list[atomicAdd(fail_count, 1u)] = j;
    }
    __syncwarp();
  }
}

// exact scores of one query row against every column (self excluded)
__global__ void k_exact_row(const float* __restrict__ wn, uint32_t n, uint32_t d, uint32_t j,
                            uint32_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float s = i == j ? -INFINITY : exact_dot(wn + (uint64_t)j * d, wn + (uint64_t)i * d, d);
    if (s == 0.0f) s = 0.0f;  // -0 == +0 under `better`: one key
    const uint32_t u = __float_as_uint(s);
    keys[i] = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    idx[i] = i;
  }
}

__global__ void k_write_row(const uint32_t* __restrict__ sorted_idx, uint32_t j, uint32_t k,
                            uint32_t* __restrict__ out) {
  for (uint32_t e = threadIdx.x; e < k; e += blockDim.x)
    out[(uint64_t)j * k + e] = e == 0 ? j : sorted_idx[e - 1];
}

}  // namespace

// Exact rows by full scans (the certificate's fallback, and the whole graph for small N / D).
static cudaError_t exact_rows(const float* wn, uint32_t n, uint32_t d, uint32_t k,
                              const uint32_t* rows, uint32_t nrows, uint32_t* out,
                              cudaStream_t s) {
  uint32_t *keys = nullptr, *idx = nullptr, *keys2 = nullptr, *idx2 = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cudaError_t e = cudaSuccess;
  e = cudaMalloc(&keys, (size_t)n * 16);
  if (e != cudaSuccess) return e;
  idx = keys + n;
  keys2 = keys + 2 * (size_t)n;
  idx2 = keys + 3 * (size_t)n;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, keys, keys2, idx, idx2, (int)n, 0, 32, s);
  e = cudaMalloc(&tmp, tb);
  for (uint32_t r = 0; r < nrows && e == cudaSuccess; ++r) {
    const uint32_t j = rows ? rows[r] : r;
    k_exact_row<<<grid_for(n, 256), 256, 0, s>>>(wn, n, d, j, keys, idx);
    size_t t2 = tb;
    e = cub::DeviceRadixSort::SortPairsDescending(tmp, t2, keys, keys2, idx, idx2, (int)n, 0, 32, s);
    if (e == cudaSuccess) k_write_row<<<1, 128, 0, s>>>(idx2, j, k, out);
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  cudaStreamSynchronize(s);
  cudaFree(tmp);
  cudaFree(keys);
  return e;
}

xknn_status_t graph_bruteforce(const float* wn, uint64_t n64, uint64_t d64, uint32_t k,
                               uint32_t kprime, uint32_t* out, cudaStream_t s,
                               uint64_t* uncertified) {
  const uint32_t n = (uint32_t)n64, d = (uint32_t)d64;
  if (k > n64) return fail_msg(XKNN_ERR_K_TOO_LARGE, "build_graph_bruteforce: k exceeds class count");
  if (k == 0) return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "build_graph_bruteforce: k must be positive");
  if (d % 4) return fail_msg(XKNN_ERR_SHAPE_MISMATCH, "dim must be a multiple of 4");
  if (uncertified) *uncertified = 0;
  cudaError_t e;
  if (d != 512 || n < 1024) {  // exact scans only
    e = exact_rows(wn, n, d, k, nullptr, n, out, s);
    return e == cudaSuccess ? XKNN_OK : fail_msg(XKNN_ERR_CUDA, cudaGetErrorString(e));
  }
  kprime = std::max<uint32_t>(kprime, k + 16);
  const uint32_t ch = (2 * kprime + 31) / 32 * 32;  // region capacity > kprime
  const uint32_t npad = (n + 255) / 256 * 256;
  __nv_bfloat16* wb = nullptr;
  float2* cand = nullptr;
  uint32_t *cnt = nullptr, *fails = nullptr;
  float* tau = nullptr;
  uint32_t nfail = 0;
  std::vector<uint32_t> flist;
#define G_CUDA(x)                                     \
  do {                                                \
    e = (x);                                          \
    if (e != cudaSuccess) goto done;                  \
  } while (0)
  G_CUDA(cudaMalloc(&wb, (size_t)npad * 512 * 2));
  G_CUDA(cudaMalloc(&cand, (size_t)npad * 2 * ch * sizeof(float2)));
  G_CUDA(cudaMalloc(&cnt, (size_t)npad * 2 * 4));
  G_CUDA(cudaMalloc(&tau, (size_t)npad * 2 * 4));
  G_CUDA(cudaMalloc(&fails, ((size_t)n + 1) * 4));
  G_CUDA(cudaMemsetAsync(fails, 0, 4, s));
  k_to_bf16<<<grid_for((uint64_t)npad * 256, 256), 256, 0, s>>>(wn, n, npad, 512, wb);
  G_CUDA(cudaGetLastError());
  G_CUDA(launch_graph_candidates(wb, n, npad, cand, cnt, tau, ch, kprime, s));
  if (getenv("XKNN_GRAPH_DEBUG")) {
    G_CUDA(cudaStreamSynchronize(s));
    std::vector<uint32_t> hc(2 * (size_t)npad);
    std::vector<float> ht(2 * (size_t)npad);
    std::vector<float2> hcand(2 * (size_t)ch);
    cudaMemcpy(hc.data(), cnt, hc.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ht.data(), tau, ht.size() * 4, cudaMemcpyDeviceToHost);
    for (uint32_t j : {0u, 1u, 300u, n - 1}) {
      cudaMemcpy(hcand.data(), cand + (size_t)j * 2 * ch, hcand.size() * 8, cudaMemcpyDeviceToHost);
      fprintf(stderr, "row %u: cnt %u %u tau %g %g :", j, hc[2 * j], hc[2 * j + 1], ht[2 * j],
              ht[2 * j + 1]);
      for (uint32_t e = 0; e < 6 && e < hc[2 * j]; ++e)
        { uint32_t ui; memcpy(&ui, &hcand[e].y, 4); fprintf(stderr, " (%u %.4f)", ui, hcand[e].x); }
      fprintf(stderr, "\n");
    }
  }
  {
    uint32_t cap = 1;
    while (cap < 2 * ch) cap <<= 1;
    const uint32_t warps = 4;
    const size_t smem = (size_t)warps * cap * 8;
    if (smem > 48 * 1024)
      G_CUDA(cudaFuncSetAttribute(k_graph_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    k_graph_finalize<<<grid_for((uint64_t)n * 32, warps * 32, 148u * 32u), warps * 32, smem, s>>>(
        wn, n, 512, cand, cnt, tau, ch, k, out, fails, fails + 1);
    G_CUDA(cudaGetLastError());
  }
  G_CUDA(cudaMemcpyAsync(&nfail, fails, 4, cudaMemcpyDeviceToHost, s));
  G_CUDA(cudaStreamSynchronize(s));
  if (nfail) {
    flist.resize(nfail);
    G_CUDA(cudaMemcpy(flist.data(), fails + 1, (size_t)nfail * 4, cudaMemcpyDeviceToHost));
    G_CUDA(exact_rows(wn, n, 512, k, flist.data(), nfail, out, s));
  }
  if (uncertified) *uncertified = nfail;
done:
#undef G_CUDA
  cudaStreamSynchronize(s);
  cudaFree(wb);
  cudaFree(cand);
  cudaFree(cnt);
  cudaFree(tau);
  cudaFree(fails);
  if (e != cudaSuccess) return fail_msg(XKNN_ERR_CUDA, cudaGetErrorString(e));
  return XKNN_OK;
}

}  // namespace xknn

extern "C" xknn_status_t xknn_graph_bruteforce(const float* w_norm_dev, uint64_t num_classes,
                                               uint64_t dim, uint32_t k, uint32_t kprime,
                                               uint32_t* out_dev, void* stream,
                                               uint64_t* uncertified_rows) {
  return xknn::graph_bruteforce(w_norm_dev, num_classes, dim, k, kprime, out_dev,
                                static_cast<cudaStream_t>(stream), uncertified_rows);
}
