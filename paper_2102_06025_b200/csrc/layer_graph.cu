// layer_graph.cu -- the layer's KNN class graph lifecycle on device:
//   xknn_layer_rebuild_graph : l2_normalize_rows of the weight shard (matrix.cpp:12-29, the
//                              reference's sequential fp64 sum), the sharded exact graph build
//                              (graph.cu; build_graph_ring, knn_graph.cpp:147-233), then
//   xknn_layer_set_graph_rows: compress_graph (knn_graph.cpp:235-266) of the row-distributed
//                              graph: every rank holds rows [begin, end) x k of the full graph;
//                              entries are bucketed by the shard that owns them and exchanged
//                              all-to-all over NCCL, so shard s receives, for every class c in
//                              rank (= class) order, the neighbours of c inside [begin_s, end_s)
//                              in their original order -- exactly CompressedKnnGraph_s;
//   xknn_layer_get_graph     : the installed CompressedKnnGraph (knn_graph.hpp:46-55).
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "graph.cuh"
#include "kernels.cuh"

namespace xknn {
namespace {

// ShardLayout::shard_of (knn_graph.cpp:94-100)
__device__ __forceinline__ uint32_t shard_of(uint64_t cls, uint64_t n, uint32_t p) {
  const uint64_t base = n / p, rem = n % p, big = rem * (base + 1);
  if (cls < big) return (uint32_t)(cls / (base + 1));
  return (uint32_t)(rem + (cls - big) / base);
}

// l2_normalize_rows_cached bit for bit: the squared norm is summed in fp64 in column order by
// one lane (the row staged in shared memory by the whole warp), norm = float(sqrt), x * (1/norm)
__global__ void k_normalize_rows_seq(const float* __restrict__ in, uint64_t rows, uint32_t d,
                                     float* __restrict__ out, unsigned long long* err) {
  extern __shared__ float srow[];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* row = srow + (uint64_t)w * d;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const float* src = in + r * d;
    for (uint32_t j = lane; j < d; j += 32) row[j] = src[j];
    __syncwarp();
    float norm = 0.f;
    if (lane == 0) {
      double sq = 0.0;
      for (uint32_t j = 0; j < d; ++j) sq += (double)row[j] * row[j];
      norm = (float)sqrt(sq);
    }
    norm = __shfl_sync(XKNN_FULL_MASK, norm, 0);
    if (norm < 1e-12f) {
      if (lane == 0) raise_error(err, XKNN_ERR_ZERO_NORM_ROW, r);
    } else {
      const float inv = 1.0f / norm;
      for (uint32_t j = lane; j < d; j += 32) out[r * d + j] = __fmul_rn(row[j], inv);
    }
    __syncwarp();
  }
}

// cnt[s][j] = neighbours of own row j owned by shard s
__global__ void k_comp_count(const uint32_t* __restrict__ rows, uint32_t n, uint32_t k,
                             uint64_t n_total, uint32_t p, uint32_t* __restrict__ cnt,
                             unsigned long long* err) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t* r = rows + (uint64_t)j * k;
    for (uint32_t s = 0; s < p; ++s) cnt[(uint64_t)s * n + j] = 0;
    for (uint32_t t = 0; t < k; ++t) {
      const uint32_t nb = r[t];
      if (nb >= n_total) {
        raise_error(err, XKNN_ERR_SHAPE_MISMATCH, j);
        continue;
      }
      ++cnt[(uint64_t)shard_of(nb, n_total, p) * n + j];
    }
  }
}

// entries bucketed by owning shard, class order inside each bucket, original order per class
__global__ void k_comp_scatter(const uint32_t* __restrict__ rows, uint32_t n, uint32_t k,
                               uint64_t n_total, uint32_t p, const uint64_t* __restrict__ pos,
                               uint32_t* __restrict__ send) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t* r = rows + (uint64_t)j * k;
    for (uint32_t s = 0; s < p; ++s) {
      uint64_t o = pos[(uint64_t)s * n + j];
      for (uint32_t t = 0; t < k; ++t) {
        const uint32_t nb = r[t];
        if (nb < n_total && shard_of(nb, n_total, p) == s) send[o++] = nb;
      }
    }
  }
}

// classify: the global winner of each query from every rank's (score, id) -- higher score,
// then lower class id (shards own ascending class ranges)
__global__ void k_merge_top1(const float2* __restrict__ all, uint32_t nq, uint32_t world,
                             uint32_t* __restrict__ out_class, float* __restrict__ out_score) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nq; j += gridDim.x * blockDim.x) {
    float bs = -INFINITY;
    uint32_t bi = 0xffffffffu;
    for (uint32_t r = 0; r < world; ++r) {
      const float2 v = all[(uint64_t)r * nq + j];
      const uint32_t id = __float_as_uint(v.y);
      if (v.x > bs || (v.x == bs && id < bi)) {
        bs = v.x;
        bi = id;
      }
    }
    out_class[j] = bi;
    if (out_score) out_score[j] = bs;
  }
}

__global__ void k_pack_top1(const float* __restrict__ sc, const uint32_t* __restrict__ id,
                            uint32_t nq, float2* __restrict__ out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nq; j += gridDim.x * blockDim.x)
    out[j] = make_float2(sc[j], __uint_as_float(id[j]));
}

}  // namespace
}  // namespace xknn

using xknn::Layer;

#define LG_CUDA(x)                                                          \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) return L.cuda_ok(e_, __FILE__, __LINE__, #x);    \
  } while (0)
#define LG_NCCL(x)                                \
  do {                                            \
    ncclResult_t r_ = (x);                        \
    if (r_ != ncclSuccess) return L.nccl_ok(r_);  \
  } while (0)

namespace {
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

xknn_status_t check_device_error(Layer& L) {
  unsigned long long w = 0;
  LG_CUDA(cudaMemcpyAsync(&w, L.err, 8, cudaMemcpyDeviceToHost, L.stream));
  LG_CUDA(cudaStreamSynchronize(L.stream));
  if (!w) return XKNN_OK;
  LG_CUDA(cudaMemsetAsync(L.err, 0, 8, L.stream));
  LG_CUDA(cudaStreamSynchronize(L.stream));
  const xknn_status_t code = (xknn_status_t)(w & 0xff);
  const std::string msg = std::string(xknn_status_string(code)) + " (device, index " +
                          std::to_string(w >> 8) + ")";
  return xknn::fail_row(code, msg.c_str(), w >> 8);
}
}  // namespace

extern "C" {

xknn_status_t xknn_layer_set_graph_rows(xknn_layer_t* h, const uint32_t* rows_dev, uint32_t k) {
  if (!h) return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "null layer handle");
  Layer& L = h->L;
  if (k == 0) return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "graph rows: k must be positive");
  const uint32_t n = (uint32_t)L.nw, p = (uint32_t)L.world;
  const uint64_t N = L.n;
  Scratch mem;
  uint32_t *cnt = nullptr, *send = nullptr, *kpc = nullptr, *flat = nullptr;
  uint64_t *pos = nullptr, *off = nullptr, *tot = nullptr;
  LG_CUDA(mem.get(&cnt, (uint64_t)p * n));
  LG_CUDA(mem.get(&pos, (uint64_t)p * n + 1));
  xknn::k_comp_count<<<xknn::grid_for(n, 256), 256, 0, L.stream>>>(rows_dev, n, k, N, p, cnt, L.err);
  LG_CUDA(cudaGetLastError());
  {
    size_t tb = 0;
    void* tmp = nullptr;
    LG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, pos, (uint64_t)p * n, L.stream));
    LG_CUDA(mem.get(reinterpret_cast<uint8_t**>(&tmp), tb));
    LG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, pos, (uint64_t)p * n, L.stream));
  }
  xknn_status_t st = check_device_error(L);
  if (st != XKNN_OK) return st;
  // per-destination totals: bucket s spans pos[s*n] .. pos[(s+1)*n] (last: + its count)
  std::vector<uint64_t> bound(p + 1);
  for (uint32_t s = 0; s < p; ++s)
    LG_CUDA(cudaMemcpyAsync(&bound[s], pos + (uint64_t)s * n, 8, cudaMemcpyDeviceToHost, L.stream));
  uint32_t lastc = 0;
  uint64_t lastp = 0;
  LG_CUDA(cudaMemcpyAsync(&lastc, cnt + (uint64_t)p * n - 1, 4, cudaMemcpyDeviceToHost, L.stream));
  LG_CUDA(cudaMemcpyAsync(&lastp, pos + (uint64_t)p * n - 1, 8, cudaMemcpyDeviceToHost, L.stream));
  LG_CUDA(cudaStreamSynchronize(L.stream));
  bound[p] = lastp + lastc;
  LG_CUDA(mem.get(&send, bound[p]));
  xknn::k_comp_scatter<<<xknn::grid_for(n, 256), 256, 0, L.stream>>>(rows_dev, n, k, N, p, pos,
                                                                     send);
  LG_CUDA(cudaGetLastError());
  // all ranks' per-destination totals: tot[r * p + s] = entries rank r sends to shard s
  LG_CUDA(mem.get(&tot, (uint64_t)p * p));
  std::vector<uint64_t> mine(p), all((uint64_t)p * p);
  for (uint32_t s = 0; s < p; ++s) mine[s] = bound[s + 1] - bound[s];
  LG_CUDA(cudaMemcpyAsync(tot + (uint64_t)L.rank * p, mine.data(), 8ull * p, cudaMemcpyHostToDevice,
                          L.stream));
  if (p > 1)
    LG_NCCL(ncclAllGather(tot + (uint64_t)L.rank * p, tot, p, ncclUint64, L.comm, L.stream));
  LG_CUDA(cudaMemcpyAsync(all.data(), tot, 8ull * p * p, cudaMemcpyDeviceToHost, L.stream));
  LG_CUDA(cudaStreamSynchronize(L.stream));
  uint64_t flat_len = 0;
  std::vector<uint64_t> rbase(p);
  for (uint32_t r = 0; r < p; ++r) {
    rbase[r] = flat_len;
    flat_len += all[(uint64_t)r * p + L.rank];
  }
  LG_CUDA(mem.get(&kpc, N));
  LG_CUDA(mem.get(&flat, flat_len));
  LG_CUDA(mem.get(&off, N));
  if (p > 1) {
    LG_NCCL(ncclGroupStart());
    for (uint32_t s = 0; s < p; ++s) {
      uint64_t sb, se;
      xknn_shard_range(N, p, s, &sb, &se);
      // my rows' per-class counts for shard s -> s; shard s's rows' counts for me <- s
      LG_NCCL(ncclSend(cnt + (uint64_t)s * n, n, ncclUint32, (int)s, L.comm, L.stream));
      LG_NCCL(ncclRecv(kpc + sb, se - sb, ncclUint32, (int)s, L.comm, L.stream));
      if (mine[s]) LG_NCCL(ncclSend(send + bound[s], mine[s], ncclUint32, (int)s, L.comm, L.stream));
      const uint64_t in = all[(uint64_t)s * p + L.rank];
      if (in) LG_NCCL(ncclRecv(flat + rbase[s], in, ncclUint32, (int)s, L.comm, L.stream));
    }
    LG_NCCL(ncclGroupEnd());
  } else {
    LG_CUDA(cudaMemcpyAsync(kpc, cnt, (uint64_t)n * 4, cudaMemcpyDeviceToDevice, L.stream));
    if (flat_len)
      LG_CUDA(cudaMemcpyAsync(flat, send, flat_len * 4, cudaMemcpyDeviceToDevice, L.stream));
  }
  {
    size_t tb = 0;
    void* tmp = nullptr;
    LG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, kpc, off, N, L.stream));
    LG_CUDA(mem.get(reinterpret_cast<uint8_t**>(&tmp), tb));
    LG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, kpc, off, N, L.stream));
  }
  L.launches += 4;
  return xknn_layer_set_graph_csr(h, kpc, off, flat, flat_len, 1);
}

xknn_status_t xknn_layer_rebuild_graph(xknn_layer_t* h, uint32_t k, uint32_t kprime,
                                       uint32_t* rows_out_dev, uint64_t* uncertified_rows) {
  if (!h) return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "null layer handle");
  Layer& L = h->L;
  if (!L.has_weights) return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "rebuild_graph: weights not set");
  if (k > L.n) return xknn::fail_msg(XKNN_ERR_K_TOO_LARGE, "build_graph: k exceeds class count");
  if (k == 0) return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "build_graph: k must be positive");
  Scratch mem;
  float* wn = nullptr;
  uint32_t* rows = nullptr;
  LG_CUDA(mem.get(&wn, L.nw * L.d));
  const unsigned threads = 256;
  const size_t smem = (threads / 32) * L.d * sizeof(float);
  if (smem > 48 * 1024)
    LG_CUDA(cudaFuncSetAttribute(xknn::k_normalize_rows_seq,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  xknn::k_normalize_rows_seq<<<xknn::grid_for(L.nw * 32, threads), threads, smem, L.stream>>>(
      L.W, L.nw, (uint32_t)L.d, wn, L.err);
  LG_CUDA(cudaGetLastError());
  ++L.launches;
  // every rank learns whether any shard hit ZeroNormRow before the collective build starts
  xknn_status_t st = check_device_error(L);
  if (L.world > 1) {
    int* flag = nullptr;
    LG_CUDA(mem.get(&flag, 1));
    int hf = st == XKNN_OK ? 0 : 1;
    LG_CUDA(cudaMemcpyAsync(flag, &hf, 4, cudaMemcpyHostToDevice, L.stream));
    LG_NCCL(ncclAllReduce(flag, flag, 1, ncclInt32, ncclMax, L.comm, L.stream));
    LG_CUDA(cudaMemcpyAsync(&hf, flag, 4, cudaMemcpyDeviceToHost, L.stream));
    LG_CUDA(cudaStreamSynchronize(L.stream));
    if (st != XKNN_OK) return st;
    if (hf) return xknn::fail_msg(XKNN_ERR_ZERO_NORM_ROW, "ZeroNormRow on another shard");
  } else if (st != XKNN_OK) {
    return st;
  }
  LG_CUDA(mem.get(&rows, L.nw * k));
  xknn::GraphBuildStats gs{};
  st = xknn::graph_build(wn, L.n, L.d, k, kprime, L.rank, L.world, L.comm, L.stream, rows, &gs);
  if (st != XKNN_OK) return st;
  if (uncertified_rows) *uncertified_rows = gs.uncertified_rows;
  if (rows_out_dev)
    LG_CUDA(cudaMemcpyAsync(rows_out_dev, rows, L.nw * k * 4, cudaMemcpyDeviceToDevice, L.stream));
  return xknn_layer_set_graph_rows(h, rows, k);
}

xknn_status_t xknn_layer_classify(xknn_layer_t* h, const float* queries_dev, uint64_t n_queries,
                                  uint32_t* out_class_dev, float* out_score_dev) {
  if (!h) return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "null layer handle");
  Layer& L = h->L;
  if (!L.has_weights) return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "classify: weights not set");
  if (n_queries == 0 || n_queries >= (1ull << 31))
    return xknn::fail_msg(XKNN_ERR_SHAPE_MISMATCH, "classify: bad query count");
  const uint32_t nq = (uint32_t)n_queries, d = (uint32_t)L.d;
  Scratch mem;
  float *qn = nullptr, *wn = nullptr, *bs = nullptr;
  uint32_t* bi = nullptr;
  float2 *mine = nullptr, *all = nullptr;
  LG_CUDA(mem.get(&qn, (uint64_t)nq * d));
  LG_CUDA(mem.get(&wn, L.nw * d));
  LG_CUDA(mem.get(&bs, nq));
  LG_CUDA(mem.get(&bi, nq));
  const unsigned threads = 256;
  const size_t smem = (threads / 32) * L.d * sizeof(float);
  if (smem > 48 * 1024)
    LG_CUDA(cudaFuncSetAttribute(xknn::k_normalize_rows_seq,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // l2_normalize_rows of the queries and of this shard's class weights, bit-exact
  xknn::k_normalize_rows_seq<<<xknn::grid_for((uint64_t)nq * 32, threads), threads, smem,
                               L.stream>>>(queries_dev, nq, d, qn, L.err);
  LG_CUDA(cudaGetLastError());
  xknn_status_t st = check_device_error(L);
  if (st != XKNN_OK) return st;
  xknn::k_normalize_rows_seq<<<xknn::grid_for(L.nw * 32, threads), threads, smem, L.stream>>>(
      L.W, L.nw, d, wn, L.err);
  LG_CUDA(cudaGetLastError());
  L.launches += 2;
  st = check_device_error(L);
  if (st != XKNN_OK) return st;
  uint64_t unc = 0;
  st = xknn::retrieval_top1_local(qn, nq, wn, (uint32_t)L.nw, (uint32_t)L.begin, d, L.stream, bs,
                                  bi, &unc);
  if (st != XKNN_OK) return st;
  LG_CUDA(mem.get(&mine, nq));
  LG_CUDA(mem.get(&all, (uint64_t)nq * L.world));
  xknn::k_pack_top1<<<xknn::grid_for(nq, 256), 256, 0, L.stream>>>(bs, bi, nq, mine);
  if (L.world > 1)
    LG_NCCL(ncclAllGather(mine, all, 2ull * nq, ncclFloat, L.comm, L.stream));
  else
    LG_CUDA(cudaMemcpyAsync(all, mine, 8ull * nq, cudaMemcpyDeviceToDevice, L.stream));
  xknn::k_merge_top1<<<xknn::grid_for(nq, 256), 256, 0, L.stream>>>(all, nq, (uint32_t)L.world,
                                                                    out_class_dev, out_score_dev);
  LG_CUDA(cudaGetLastError());
  L.launches += 2;
  LG_CUDA(cudaStreamSynchronize(L.stream));
  return XKNN_OK;
}

xknn_status_t xknn_layer_get_graph(xknn_layer_t* h, uint32_t* k_per_class, uint64_t* offsets,
                                   uint32_t* flat, uint64_t flat_capacity, uint64_t* flat_len,
                                   int on_device) {
  if (!h) return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "null layer handle");
  Layer& L = h->L;
  if (!L.has_graph) return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "no graph installed");
  if (flat_len) *flat_len = L.g_flat_len;
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (k_per_class) LG_CUDA(cudaMemcpyAsync(k_per_class, L.g_kpc, L.n * 4, kind, L.stream));
  if (offsets) LG_CUDA(cudaMemcpyAsync(offsets, L.g_off, L.n * 8, kind, L.stream));
  if (flat) {
    if (flat_capacity < L.g_flat_len)
      return xknn::fail_msg(XKNN_ERR_SHAPE_MISMATCH, "get_graph: flat capacity too small");
    if (L.g_flat_len) LG_CUDA(cudaMemcpyAsync(flat, L.g_flat, L.g_flat_len * 4, kind, L.stream));
  }
  LG_CUDA(cudaStreamSynchronize(L.stream));
  return XKNN_OK;
}

}  // extern "C"
