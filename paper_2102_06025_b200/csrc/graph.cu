// graph.cu -- exact KNN class graph on device, sharded over the class blocks of P GPUs:
// build_graph_ring (knn_graph.cpp:147-233) and, at P = 1, build_graph_bruteforce (:124-145),
// under the reference's ordering `better` (:20-26): self first, then descending inner product
// (fp32, ascending d, separate multiply and add: matrix.cpp:57-68 / knn_graph.cpp:137-138),
// ties to the lower class index.  Bit-exact with the reference:
//   1. candidate ring (fp16 tensor cores): every rank scores its own normalized rows against
//      each class block as it passes around the ring (ncclSend/Recv to rank+1, P-1 hops, the
//      reference's rotation held[(s+1)%p] = held[s]); a threshold top-k' epilogue of the GEMM
//      (fast.cu, k_gemm2<kG>) keeps per row a list of at most k' candidates and a cut T: every
//      column left out has approximate score <= T;
//   2. certificate + window: with A = the (k-1)-th largest approximate score in the list and
//      eps >= |approx - reference fp32 score|, the row is certified when A > T + 2 eps (its
//      k-1 best exact scores then beat every left-out column); only list entries with approx
//      >= A - 2 eps can reach the exact top k-1, the others are dropped;
//   3. exact ring (fp32): the blocks pass around once more and each rank re-scores its
//      windows' candidates in the reference's arithmetic as their block goes by; rows that
//      failed the certificate are scanned exactly against every block instead;
//   4. finalize: sort under `better`, self first, keep k.
// compress_graph (knn_graph.cpp:235-266) of the row-distributed result is an all-to-all of
// graph entries by owning shard (xknn_layer_rebuild_graph, layer_graph.cu).
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <vector>

#include "graph.cuh"
#include "kernels.cuh"

namespace xknn {

cudaError_t launch_graph_candidates(const __half* own, uint32_t nrows, uint32_t row_base,
                                    const __half* held, uint32_t ncols, uint32_t col_base,
                                    float2* list, uint32_t* lcnt, float* lcut, uint32_t kprime,
                                    uint32_t kcap, float2* cand, uint32_t* cnt, float* tau,
                                    uint32_t ch, cudaStream_t s);

namespace {

// |fp16 tensor-core score - reference fp32 score| for unit rows at D = 512: input rounding
// 2 * 2^-11 (+ subnormal terms 2e-6), fp32 accumulation of 512 products (512 * 2^-23), the
// reference's own sequential fp32 sum (512 * 2^-24 + 2^-24); 1.07e-3 in total, with margin:
constexpr float kEps = 0.00125f;
constexpr size_t kRescoreSmem = 8 * (512 + 32 * 33) * sizeof(float);  // 8 warps per block

__global__ void k_to_f16(const float* __restrict__ w, uint64_t n, uint64_t npad, uint32_t d,
                         __half* __restrict__ out) {
  const uint64_t total = npad * d / 2;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = (2 * e) / d;
    float2 v = row < n ? reinterpret_cast<const float2*>(w)[e] : make_float2(0.f, 0.f);
    reinterpret_cast<__half2*>(out)[e] = __floats2half2_rn(v.x, v.y);
  }
}

// every stride-th own row (fp16) -> a pilot block of ns rows (zero rows up to a multiple of 256)
__global__ void k_sample_rows(const __half* __restrict__ own, uint32_t stride, uint32_t ns,
                              uint32_t nspad, __half* __restrict__ out) {
  const uint64_t total = (uint64_t)nspad * 64;  // 16-B units, 64 per 512-wide row
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = e / 64, c = e % 64;
    reinterpret_cast<uint4*>(out)[e] =
        r < ns ? reinterpret_cast<const uint4*>(own)[(r * stride) * 64 + c] : make_uint4(0, 0, 0, 0);
  }
}

__global__ void k_list_init(uint32_t* lcnt, float* lcut, uint64_t n) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    lcnt[j] = 0;
    lcut[j] = -INFINITY;
  }
}

__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float funkey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
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

// Pilot seed, one warp per row: after the pilot pass against a strided sample of all classes,
// the row's cut starts at the j-th best approximate sample score (the list is emptied; every
// column is scanned again by the main pass).  A cut is only ever a bound on what was left out,
// so any starting value is correct; a too-high one shows up as an uncertified row (exact
// fallback).  With 1 in `stride` columns sampled, the seed lies above the row's (k-1)-th best
// + 2 eps (about its 125th best on random unit rows) only if j of those fell in the sample:
// a Poisson(125 / 32) tail, ~1e-7 at j = 18.  The seed sits near the row's j*stride-th best,
// so the main pass inserts few more than k' entries per row.
__global__ void k_seed_cut(const float2* __restrict__ list, uint32_t* __restrict__ lcnt,
                           float* __restrict__ lcut, uint32_t n, uint32_t kc, uint32_t j) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n;
       r += (gridDim.x * blockDim.x) >> 5) {
    const float2* L = list + (uint64_t)r * kc;
    const uint32_t m = lcnt[r];
    float seed = -INFINITY;
    if (m >= j) {  // j-th largest: largest key with #(>= key) >= j
      uint32_t lo = 0, hi = 0xffffffffu;
      while (lo < hi) {
        const uint32_t mid = (uint32_t)(((uint64_t)lo + hi + 1) >> 1);
        uint32_t c = 0;
        for (uint32_t e = lane; e < m; e += 32) c += fkey(L[e].x) >= mid;
        c = warp_sum(c);
        if (c >= j) lo = mid; else hi = mid - 1;
      }
      seed = funkey(lo);
    }
    __syncwarp();
    if (lane == 0) {
      lcnt[r] = 0;
      lcut[r] = seed;
    }
  }
}

// Step 2, one warp per row: certificate and candidate window (see the file comment).
__global__ void k_window(float2* __restrict__ list, uint32_t* __restrict__ lcnt,
                         const float* __restrict__ lcut, uint32_t n, uint32_t kc, uint32_t need,
                         uint32_t* __restrict__ flag, uint32_t* __restrict__ unc_count,
                         uint32_t* __restrict__ unc_list) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n;
       j += (gridDim.x * blockDim.x) >> 5) {
    float2* L = list + (uint64_t)j * kc;
    const uint32_t m = lcnt[j];
    const float T = lcut[j];
    bool cert = false;
    float theta = -INFINITY;
    if (m >= need) {
      // A = need-th largest approximate score: largest key with #(>= key) >= need
      uint32_t lo = 0, hi = 0xffffffffu;
      while (lo < hi) {
        const uint32_t mid = (uint32_t)(((uint64_t)lo + hi + 1) >> 1);
        uint32_t c = 0;
        for (uint32_t e = lane; e < m; e += 32) c += fkey(L[e].x) >= mid;
        c = warp_sum(c);
        if (c >= need) lo = mid; else hi = mid - 1;
      }
      const float A = funkey(lo);
      cert = (T == -INFINITY) || (A > T + 2.0f * kEps);  // T = -inf: every column is listed
      theta = A - 2.0f * kEps;
    }
    if (cert) {
      uint32_t w = 0;
      for (uint32_t base = 0; base < m; base += 32) {
        const uint32_t e = base + lane;
        const float2 v = e < m ? L[e] : make_float2(-INFINITY, 0.f);
        const bool keep = e < m && v.x >= theta;
        __syncwarp();
        const uint32_t bal = __ballot_sync(XKNN_FULL_MASK, keep);
        if (keep) L[w + __popc(bal & ((1u << lane) - 1))] = v;
        w += __popc(bal);
        __syncwarp();
      }
      if (lane == 0) {
        lcnt[j] = w;
        flag[j] = 0;
      }
    } else if (lane == 0) {
      const uint32_t u = atomicAdd(unc_count, 1u);
      unc_list[u] = j;
      flag[j] = u + 1;
    }
    __syncwarp();
  }
}

// Step 3, one warp per own row: exact scores of the window entries that live in the held block
// [cb, cb + nc) (fp32 rows `held`).  ex[row][e] parallels list[row][e].
__global__ void k_rescore(const float* __restrict__ own, uint32_t n, uint32_t d,
                          const float2* __restrict__ list, const uint32_t* __restrict__ lcnt,
                          const uint32_t* __restrict__ flag, uint32_t kc,
                          const float* __restrict__ held, uint32_t cb, uint32_t nc,
                          float* __restrict__ ex) {
  // D = 512.  Lane l carries candidate l of a group of 32 through the reference's sequential
  // sum; the 32 candidate rows stream through shared memory in 128-B column chunks loaded by
  // the whole warp (four row segments per instruction) instead of 32 scattered row walks.
  extern __shared__ float rs_smem[];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* qrow = rs_smem + (uint64_t)w * (512 + 32 * 33);  // the own row
  float* stg = qrow + 512;                                // 32 rows x 32 floats (+1 pad)
  for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n;
       j += (gridDim.x * blockDim.x) >> 5) {
    if (flag[j]) continue;
    const uint32_t m = lcnt[j];
    const float2* L = list + (uint64_t)j * kc;
    __syncwarp();
    for (uint32_t c = lane; c < 128; c += 32)
      reinterpret_cast<float4*>(qrow)[c] = reinterpret_cast<const float4*>(own + (uint64_t)j * 512)[c];
    for (uint32_t base = 0; base < m; base += 32) {
      const uint32_t e = base + lane;
      const uint32_t id = e < m ? __float_as_uint(L[e].y) : 0xffffffffu;
      const bool mine = e < m && id - cb < nc;
      const uint32_t act = __ballot_sync(XKNN_FULL_MASK, mine);
      if (!act) continue;
      const uint64_t rbase = mine ? (uint64_t)(id - cb) * 512 : 0;
      float acc = 0.0f;
      for (uint32_t c = 0; c < 16; ++c) {  // 32-column chunk c of every candidate row
        __syncwarp();
#pragma unroll
        for (uint32_t i = 0; i < 8; ++i) {
          const uint32_t r = 4 * i + (lane >> 3);  // row (candidate lane) of this load
          const uint64_t rb = __shfl_sync(XKNN_FULL_MASK, rbase, r);
          const bool on = (act >> r) & 1u;
          const float4 v = on ? reinterpret_cast<const float4*>(held + rb + c * 32)[lane & 7]
                              : make_float4(0.f, 0.f, 0.f, 0.f);
          float* dst = stg + r * 33 + (lane & 7) * 4;
          dst[0] = v.x;
          dst[1] = v.y;
          dst[2] = v.z;
          dst[3] = v.w;
        }
        __syncwarp();
        const float* mine_row = stg + lane * 33;
        const float* q = qrow + c * 32;
#pragma unroll
        for (uint32_t t = 0; t < 32; ++t) acc = __fadd_rn(acc, __fmul_rn(q[t], mine_row[t]));
      }
      if (mine) ex[(uint64_t)j * kc + e] = acc;
    }
  }
}

// ---- batched exact top-`need` of query rows against a block (rows whose fp16 certificate
// failed, classify queries, the D != 512 path).  Per batch of up to kXR rows: every row's
// exact keys against the block (the reference's dot order), then a 4-pass 8-bit radix select
// per row for the `need`-th best key T, then the keys above T plus the first ties of T in column
// order (`better` breaks score ties to the lower id), sentinel-padded when the block has fewer.
// Replaces a scan + a full CUB sort per row and block.
constexpr uint32_t kXR = 16;        // query rows per batch (their rows staged in smem)
constexpr uint32_t kXChunk = 4096;  // columns per select block

struct XSel {
  uint32_t prefix, mask, rem, gtn, done;  // T's bits so far, their mask, ties still to take,
};                                        // keys above T, fewer valid keys than `need`

__global__ void k_xinit(XSel* st, uint32_t nr, uint32_t need, uint32_t* ctr) {
  const uint32_t u = threadIdx.x;
  if (u < nr) {
    st[u] = XSel{0u, 0u, need, 0u, 0u};
    ctr[u] = 0;
  }
}

// keys[u][i]: the order-preserving key of the exact score of query row rows[u] against block
// row i (0 = the query itself, self id = self_base + rows[u]; self_base = ~0: no self)
__global__ void k_xscan_rows(const float* __restrict__ q, const uint32_t* __restrict__ rows,
                             uint32_t nr, uint32_t self_base, const float* __restrict__ blk,
                             uint32_t nc, uint32_t d, uint32_t cb, uint32_t* __restrict__ keys) {
  extern __shared__ float sq[];  // nr x d
  for (uint32_t t = threadIdx.x; t < nr * d; t += blockDim.x)
    sq[t] = q[(uint64_t)rows[t / d] * d + t % d];
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    const float* col = blk + (uint64_t)i * d;
    for (uint32_t u = 0; u < nr; ++u) {
      uint32_t key = 0;
      if (self_base == 0xffffffffu || cb + i != self_base + rows[u]) {
        float sc = exact_dot(sq + (uint64_t)u * d, col, d);
        if (sc == 0.0f) sc = 0.0f;  // -0 == +0 under `better`: one key
        key = fkey(sc);
      }
      keys[(uint64_t)u * nc + i] = key;
    }
  }
}

// radix-select pass: histogram of the `shift` digit over the keys matching the prefix so far
__global__ void k_xhist(const uint32_t* __restrict__ keys, uint32_t nc, const XSel* __restrict__ st,
                        uint32_t* __restrict__ hist, uint32_t shift) {
  __shared__ uint32_t h[256];
  const uint32_t u = blockIdx.y;
  const XSel x = st[u];
  if (x.done) return;  // uniform per block
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t* k = keys + (uint64_t)u * nc;
  const uint32_t i1 = min(nc, (blockIdx.x + 1) * kXChunk);
  for (uint32_t i = blockIdx.x * kXChunk + threadIdx.x; i < i1; i += blockDim.x) {
    const uint32_t key = k[i];
    if (key != 0 && (key & x.mask) == x.prefix) atomicAdd(&h[(key >> shift) & 255u], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&hist[u * 256 + threadIdx.x], h[threadIdx.x]);
}

// ... and the digit of the rem-th best key; clears the histogram for the next pass
__global__ void k_xpick(uint32_t* __restrict__ hist, XSel* __restrict__ st, uint32_t shift,
                        uint32_t need) {
  __shared__ uint32_t h[256];
  const uint32_t u = blockIdx.x;
  h[threadIdx.x] = hist[u * 256 + threadIdx.x];
  hist[u * 256 + threadIdx.x] = 0;
  __syncthreads();
  if (threadIdx.x) return;
  XSel x = st[u];
  if (x.done) return;
  uint32_t tot = 0;
  for (int dg = 0; dg < 256; ++dg) tot += h[dg];
  if (shift == 24 && tot < x.rem) {  // fewer valid keys than `need`: take them all (T = 0)
    st[u] = XSel{0u, 0u, 0u, tot, 1u};
    return;
  }
  uint32_t above = 0;
  for (int dg = 255; dg >= 0; --dg) {
    if (above + h[dg] >= x.rem) {
      x.prefix |= (uint32_t)dg << shift;
      x.mask |= 255u << shift;
      x.rem -= above;
      break;
    }
    above += h[dg];
  }
  if (shift == 0) x.gtn = need - x.rem;
  st[u] = x;
}

// ties of T per chunk, then their exclusive prefix over the chunks (column order)
__global__ void k_xties(const uint32_t* __restrict__ keys, uint32_t nc, const XSel* __restrict__ st,
                        uint32_t* __restrict__ tiecnt, uint32_t nchunks) {
  __shared__ uint32_t c;
  const uint32_t u = blockIdx.y;
  const XSel x = st[u];
  if (threadIdx.x == 0) c = 0;
  __syncthreads();
  if (!x.done && x.rem) {
    const uint32_t* k = keys + (uint64_t)u * nc;
    const uint32_t i1 = min(nc, (blockIdx.x + 1) * kXChunk);
    uint32_t m = 0;
    for (uint32_t i = blockIdx.x * kXChunk + threadIdx.x; i < i1; i += blockDim.x)
      m += k[i] == x.prefix;
    if (m) atomicAdd(&c, m);
  }
  __syncthreads();
  if (threadIdx.x == 0) tiecnt[(uint64_t)u * nchunks + blockIdx.x] = c;
}
__global__ void k_xtiescan(uint32_t* __restrict__ tiecnt, uint32_t nchunks) {
  uint32_t* t = tiecnt + (uint64_t)blockIdx.x * nchunks;
  uint32_t run = 0;
  for (uint32_t c = 0; c < nchunks; ++c) {
    const uint32_t v = t[c];
    t[c] = run;
    run += v;
  }
}

// the keys above T (any order) and the first `rem` ties of T in column order, as (score, id)
__global__ void k_xcollect(const uint32_t* __restrict__ keys, uint32_t nc, uint32_t cb,
                           const XSel* __restrict__ st, const uint32_t* __restrict__ tieoff,
                           uint32_t nchunks, float2* __restrict__ out, uint64_t ostride,
                           uint32_t* __restrict__ ctr) {
  __shared__ uint32_t wcnt[8];
  const uint32_t u = blockIdx.y, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const XSel x = st[u];
  const uint32_t T = x.done ? 0u : x.prefix;
  const bool ties = !x.done && x.rem;
  const uint32_t* k = keys + (uint64_t)u * nc;
  float2* o = out + (uint64_t)u * ostride;
  uint32_t run = ties ? tieoff[(uint64_t)u * nchunks + blockIdx.x] : 0;
  const uint32_t i0 = blockIdx.x * kXChunk, i1 = min(nc, i0 + kXChunk);
  for (uint32_t base = i0; base < i1; base += blockDim.x) {  // uniform trip count
    const uint32_t i = base + threadIdx.x;
    const uint32_t key = i < i1 ? k[i] : 0u;
    if (key > T) o[atomicAdd(&ctr[u], 1u)] = make_float2(funkey(key), __uint_as_float(cb + i));
    if (!ties) continue;
    const bool tie = key == T && key != 0u;
    const uint32_t bal = __ballot_sync(0xffffffffu, tie);
    if (lane == 0) wcnt[w] = __popc(bal);
    __syncthreads();
    uint32_t before_w = 0, all = 0;
    for (uint32_t v = 0; v < blockDim.x / 32; ++v) {
      before_w += v < w ? wcnt[v] : 0u;
      all += wcnt[v];
    }
    if (tie) {
      const uint32_t r = run + before_w + __popc(bal & ((1u << lane) - 1u));
      if (r < x.rem) o[x.gtn + r] = make_float2(funkey(key), __uint_as_float(cb + i));
    }
    run += all;
    __syncthreads();
  }
}

// sentinel padding of rows with fewer valid keys than `need`
__global__ void k_xpad(const XSel* __restrict__ st, float2* __restrict__ out, uint64_t ostride,
                       uint32_t need) {
  const XSel x = st[blockIdx.x];
  if (!x.done) return;
  for (uint32_t e = x.gtn + threadIdx.x; e < need; e += blockDim.x)
    out[(uint64_t)blockIdx.x * ostride + e] = make_float2(-INFINITY, __uint_as_float(0xffffffffu));
}

// Step 4, one warp per row: sort the row's exactly scored candidates under `better` (warp
// bitonic in shared memory), write self + the k-1 best.
__global__ void k_finalize(uint32_t n, uint32_t row_base, uint32_t k, uint32_t kc, uint32_t cap,
                           const float2* __restrict__ list, const uint32_t* __restrict__ lcnt,
                           const float* __restrict__ ex, const uint32_t* __restrict__ flag,
                           const float2* __restrict__ ubuf, uint32_t ulen,
                           uint32_t* __restrict__ out) {
  extern __shared__ uint8_t sm[];
  const uint32_t warps = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* ss = reinterpret_cast<float*>(sm) + (uint64_t)w * cap;
  uint32_t* si = reinterpret_cast<uint32_t*>(reinterpret_cast<float*>(sm) + (uint64_t)warps * cap) +
                 (uint64_t)w * cap;
  for (uint32_t j = blockIdx.x * warps + w; j < n; j += gridDim.x * warps) {
    const uint32_t f = flag[j];
    const uint32_t m = f ? ulen : lcnt[j];
    for (uint32_t e = lane; e < cap; e += 32) {
      float s = -INFINITY;
      uint32_t i = 0xffffffffu;
      if (e < m) {
        if (f) {
          const float2 v = ubuf[(uint64_t)(f - 1) * ulen + e];
          s = v.x;
          i = __float_as_uint(v.y);
        } else {
          s = ex[(uint64_t)j * kc + e];
          i = __float_as_uint(list[(uint64_t)j * kc + e].y);
        }
      }
      ss[e] = s;
      si[e] = i;
    }
    __syncwarp();
    for (uint32_t size = 2; size <= cap; size <<= 1) {
      for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (uint32_t e = lane; e < cap; e += 32) {
          const uint32_t p = e ^ stride;
          if (p > e) {
            const bool dir = (e & size) == 0;
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
    uint32_t* o = out + (uint64_t)j * k;
    for (uint32_t e = lane; e < k; e += 32) o[e] = e == 0 ? row_base + j : si[e - 1];
    __syncwarp();
  }
}

// classify: one warp per query, the best exactly scored candidate (higher score, then lower
// class id) of its window, or its exact scan's winner when uncertified
__global__ void k_top1(uint32_t n, uint32_t kc, const float2* __restrict__ list,
                       const uint32_t* __restrict__ lcnt, const float* __restrict__ ex,
                       const uint32_t* __restrict__ flag, const float2* __restrict__ ubuf,
                       float* __restrict__ best_score, uint32_t* __restrict__ best_id) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n;
       j += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t f = flag[j];
    float bs = -INFINITY;
    uint32_t bi = 0xffffffffu;
    if (f) {
      if (lane == 0) {
        const float2 v = ubuf[f - 1];
        bs = v.x;
        bi = __float_as_uint(v.y);
      }
    } else {
      for (uint32_t e = lane; e < lcnt[j]; e += 32) {
        const float sc = ex[(uint64_t)j * kc + e];
        const uint32_t id = __float_as_uint(list[(uint64_t)j * kc + e].y);
        if (before(sc, id, bs, bi)) {
          bs = sc;
          bi = id;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float os = __shfl_xor_sync(XKNN_FULL_MASK, bs, o);
      const uint32_t oi = __shfl_xor_sync(XKNN_FULL_MASK, bi, o);
      if (before(os, oi, bs, bi)) {
        bs = os;
        bi = oi;
      }
    }
    if (lane == 0) {
      best_score[j] = bs;
      best_id[j] = bi;
    }
  }
}

__global__ void k_self_only(uint32_t n, uint32_t row_base, uint32_t* out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    out[j] = row_base + j;
}

}  // namespace


namespace {
// RAII device scratch, stream-ordered from the device's default memory pool.  Freed blocks stay
// mapped in the pool (like a caching allocator): the next build -- the layer's periodic rebuild
// -- reuses them without mapping or unmapping GBs through the driver (which costs 0.1-1 s per
// build at 1M rows).  xknn_graph_release_cache() returns them (cf. torch.cuda.empty_cache()).
struct Dev {
  cudaStream_t s;
  std::vector<void*> p;
  explicit Dev(cudaStream_t st) : s(st) {
    int dev = 0;
    cudaMemPool_t pool = nullptr;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  ~Dev() {
    for (void* q : p)
      if (q) cudaFreeAsync(q, s);
  }
  template <typename T>
  cudaError_t get(T** out, uint64_t count) {
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, std::max<uint64_t>(count, 1) * sizeof(T), s);
    if (e == cudaSuccess) p.push_back(q);
    *out = static_cast<T*>(q);
    return e;
  }
  void release(void* q) {  // after every use of q enqueued so far on s (or joined into s)
    for (auto& x : p)
      if (x == q) {
        cudaFreeAsync(x, s);
        x = nullptr;
      }
  }
};

// The `need` best (score, global id) under `better` of query rows rows_dev[0..nr) of q (d floats
// each) against blk (nc rows, global ids cb..), excluding id self_base + rows[u] (~0: none):
// out[u * ostride + e], e < need, in no particular order (k_finalize / k_top1 sort), sentinel-
// padded where the block has fewer.  Bit-identical to a full descending sort of the exact keys
// (stable on the column index) and its first `need` entries.
cudaError_t exact_topk(const float* q, const uint32_t* rows_dev, uint32_t nr, uint32_t self_base,
                       const float* blk, uint32_t nc, uint32_t d, uint32_t cb, uint32_t need,
                       float2* out, uint64_t ostride, Dev& mem, cudaStream_t s) {
  if (!nr || !need) return cudaSuccess;
  uint32_t R = std::min<uint32_t>(kXR, std::max<uint32_t>(1u, 12288u / d));  // rows in 48 KB smem
  R = std::min<uint64_t>(R, std::max<uint64_t>(1, (256ull << 20) / 4 / std::max(nc, 1u)));
  const uint32_t nchunks = (nc + kXChunk - 1) / kXChunk;
  uint32_t *keys = nullptr, *hist = nullptr, *tie = nullptr, *ctr = nullptr;
  XSel* st = nullptr;
  cudaError_t e;
  if ((e = mem.get(&keys, (uint64_t)R * nc)) != cudaSuccess) return e;
  if ((e = mem.get(&hist, (uint64_t)R * 256)) != cudaSuccess) return e;
  if ((e = mem.get(&tie, (uint64_t)R * nchunks)) != cudaSuccess) return e;
  if ((e = mem.get(&ctr, R)) != cudaSuccess) return e;
  if ((e = mem.get(&st, R)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(hist, 0, (size_t)R * 256 * 4, s)) != cudaSuccess) return e;
  const unsigned sgrid = grid_for(nc, 256, 148u * 8u);
  for (uint32_t u0 = 0; u0 < nr; u0 += R) {
    const uint32_t r = std::min(R, nr - u0);
    float2* o = out + (uint64_t)u0 * ostride;
    k_xinit<<<1, 32, 0, s>>>(st, r, need, ctr);
    k_xscan_rows<<<sgrid, 256, (size_t)r * d * 4, s>>>(q, rows_dev + u0, r, self_base, blk, nc, d,
                                                       cb, keys);
    for (int shift = 24; shift >= 0; shift -= 8) {
      k_xhist<<<dim3(nchunks, r), 256, 0, s>>>(keys, nc, st, hist, (uint32_t)shift);
      k_xpick<<<r, 256, 0, s>>>(hist, st, (uint32_t)shift, need);
    }
    k_xties<<<dim3(nchunks, r), 256, 0, s>>>(keys, nc, st, tie, nchunks);
    k_xtiescan<<<r, 1, 0, s>>>(tie, nchunks);
    k_xcollect<<<dim3(nchunks, r), 256, 0, s>>>(keys, nc, cb, st, tie, nchunks, o, ostride, ctr);
    k_xpad<<<r, 128, 0, s>>>(st, o, ostride, need);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

__global__ void k_iota_rows(uint32_t* rows, uint32_t* flag, uint32_t n) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    rows[j] = j;
    flag[j] = j + 1;
  }
}

// Exact rows by full scans at P = 1 (the whole graph for D != 512): every row's exact k-1 best
// (exact_topk), then self first + sorted by k_finalize.
cudaError_t exact_rows(const float* wn, uint32_t n, uint32_t d, uint32_t k, uint32_t* out,
                       cudaStream_t s) {
  Dev mem(s);
  const uint32_t need = k - 1;
  uint32_t *rows = nullptr, *flag = nullptr;
  float2* ubuf = nullptr;
  cudaError_t e;
  if ((e = mem.get(&rows, n)) != cudaSuccess) return e;
  if ((e = mem.get(&flag, n)) != cudaSuccess) return e;
  if ((e = mem.get(&ubuf, (uint64_t)n * need)) != cudaSuccess) return e;
  k_iota_rows<<<grid_for(n, 256), 256, 0, s>>>(rows, flag, n);
  if ((e = exact_topk(wn, rows, n, 0, wn, n, d, 0, need, ubuf, need, mem, s)) != cudaSuccess)
    return e;
  uint32_t cap = 1;
  while (cap < need) cap <<= 1;
  const uint32_t warps = 4;
  const size_t smem = (size_t)warps * cap * 8;
  if (smem > 48 * 1024 &&
      (e = cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem)) != cudaSuccess)
    return e;
  k_finalize<<<grid_for((uint64_t)n * 32, warps * 32, 148u * 32u), warps * 32, smem, s>>>(
      n, 0, k, 1, cap, nullptr, nullptr, nullptr, flag, ubuf, need, out);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

inline void shard_range_of(uint64_t n, uint64_t p, uint64_t s, uint64_t* b, uint64_t* e) {
  const uint64_t base = n / p, rem = n % p;
  if (s < rem) {
    *b = s * (base + 1);
    *e = *b + base + 1;
  } else {
    *b = rem * (base + 1) + (s - rem) * base;
    *e = *b + base;
  }
}
}  // namespace

xknn_status_t graph_build(const float* wn, uint64_t n_total, uint64_t d64, uint32_t k,
                          uint32_t kprime, int rank, int world, ncclComm_t comm, cudaStream_t s,
                          uint32_t* out, GraphBuildStats* stats) {
  if (stats) *stats = GraphBuildStats{};
  if (world < 1 || rank < 0 || rank >= world)
    return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "graph build: bad rank/world");
  if (k > n_total) return fail_msg(XKNN_ERR_K_TOO_LARGE, "build_graph: k exceeds class count");
  if (k == 0) return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "build_graph: k must be positive");
  if (d64 == 0 || d64 % 4) return fail_msg(XKNN_ERR_SHAPE_MISMATCH, "dim must be a positive multiple of 4");
  if (n_total >= (1ull << 32) - 1) return fail_msg(XKNN_ERR_UNSUPPORTED, "class ids must fit u32");
  if (n_total < (uint64_t)world) return fail_msg(XKNN_ERR_EMPTY_SHARD, "build_graph_ring: a shard is empty");
  if (world > 1 && !comm) return fail_msg(XKNN_ERR_INVALID_ARGUMENT, "graph ring: NCCL communicator required");
  const uint32_t d = (uint32_t)d64;
  const auto host_t0 = std::chrono::steady_clock::now();
  uint64_t b64, e64;
  shard_range_of(n_total, world, rank, &b64, &e64);
  const uint32_t row_base = (uint32_t)b64, n = (uint32_t)(e64 - b64);
  cudaError_t e = cudaSuccess;
#define G_CUDA(x)                                                         \
  do {                                                                    \
    e = (x);                                                              \
    if (e != cudaSuccess) return fail_msg(XKNN_ERR_CUDA, cudaGetErrorString(e)); \
  } while (0)
#define G_NCCL(x)                                                         \
  do {                                                                    \
    ncclResult_t r_ = (x);                                                \
    if (r_ != ncclSuccess) return fail_msg(XKNN_ERR_NCCL, ncclGetErrorString(r_)); \
  } while (0)
  if (k == 1) {  // self only
    k_self_only<<<grid_for(n, 256), 256, 0, s>>>(n, row_base, out);
    G_CUDA(cudaGetLastError());
    G_CUDA(cudaStreamSynchronize(s));
    return XKNN_OK;
  }
  if (d != 512) {
    if (world > 1) return fail_msg(XKNN_ERR_UNSUPPORTED, "graph ring needs dim 512");
    G_CUDA(exact_rows(wn, n, d, k, out, s));
    if (stats) stats->uncertified_rows = n;
    return XKNN_OK;
  }
  const uint32_t need = k - 1;
  // k' is a performance knob here (the output never depends on it): large enough that the
  // certificate holds for almost every row
  const uint32_t kp = std::max<uint32_t>({kprime, 2 * k, k + 32});
  // region capacity per (slot, half); 1.25-3x k' measured alike at 1M classes
  const uint32_t ch = (2 * kp + 31) / 32 * 32;
  // list capacity (row stride of list / ex): k' plus room for the appends of later column chunks
  const uint32_t kc = (kp + 48 + 31) / 32 * 32;
  uint64_t maxrows = 0;
  for (int r = 0; r < world; ++r) {
    uint64_t rb, re;
    shard_range_of(n_total, world, r, &rb, &re);
    maxrows = std::max(maxrows, re - rb);
  }
  const uint64_t npad = (n + 255) / 256 * 256, mpad = (maxrows + 255) / 256 * 256;
  Dev mem(s);
  float2 *list = nullptr, *cand = nullptr;
  uint32_t *lcnt = nullptr, *ccnt = nullptr, *flag = nullptr, *unc = nullptr;
  float *lcut = nullptr, *ctau = nullptr, *ex = nullptr;
  __half *own16 = nullptr, *buf16[2] = {nullptr, nullptr};
  G_CUDA(mem.get(&list, (uint64_t)n * kc));
  G_CUDA(mem.get(&lcnt, n));
  G_CUDA(mem.get(&lcut, n));
  G_CUDA(mem.get(&cand, (uint64_t)kNumSMs / 2 * 256 * 2 * ch));
  G_CUDA(mem.get(&ccnt, (uint64_t)kNumSMs / 2 * 256 * 2));
  G_CUDA(mem.get(&ctau, (uint64_t)kNumSMs / 2 * 256 * 2));
  G_CUDA(mem.get(&own16, npad * 512));
  if (world > 1) {
    G_CUDA(mem.get(&buf16[0], mpad * 512));
    G_CUDA(mem.get(&buf16[1], mpad * 512));
  }
  cudaStream_t cs = nullptr;
  std::vector<cudaEvent_t> evs;
  struct Cleanup {
    cudaStream_t* cs;
    std::vector<cudaEvent_t>* evs;
    ~Cleanup() {
      for (auto ev : *evs) cudaEventDestroy(ev);
      if (*cs) cudaStreamDestroy(*cs);
    }
  } cleanup{&cs, &evs};
  auto new_event = [&](cudaEvent_t* ev) {
    cudaError_t r = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (r == cudaSuccess) evs.push_back(*ev);
    return r;
  };
  if (world > 1) G_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  const int next = (rank + 1) % world, prev = (rank + world - 1) % world;

  // optional phase timing (XKNN_GRAPH_TIMING=1): candidates, window, exact ring, finalize
  const bool timing = getenv("XKNN_GRAPH_TIMING") || getenv("XKNN_GRAPH_SCAN_ONLY");
  cudaEvent_t tev[6] = {};
  if (timing)
    for (auto& ev : tev) {
      G_CUDA(cudaEventCreate(&ev));
      evs.push_back(ev);
    }
  if (timing) {
    G_CUDA(cudaEventRecord(tev[0], s));
    fprintf(stderr, "[xknn graph] host prologue %.2f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count());
  }
  // ---- 1. candidate ring (fp16) ----
  k_to_f16<<<grid_for(npad * 256, 256), 256, 0, s>>>(wn, n, npad, 512, own16);
  G_CUDA(cudaGetLastError());
  k_list_init<<<grid_for(n, 256), 256, 0, s>>>(lcnt, lcut, n);
  G_CUDA(cudaGetLastError());
  {
    // pilot: seed every row's cut from a 1-in-32 strided sample of ALL classes (k_seed_cut):
    // every rank samples 1 in 32*P of its block and the samples are all-gathered
    uint64_t minrows = ~0ull;
    for (int r = 0; r < world; ++r) {
      uint64_t rb, re;
      shard_range_of(n_total, world, r, &rb, &re);
      minrows = std::min(minrows, re - rb);
    }
    const uint32_t jseed = 18, stride = 32u * (uint32_t)world;
    // the pilot keeps k' = 32: small regions compact cheaply (53 vs 74 ms at 1M with 416)
    const uint32_t pilot_ch = std::min<uint32_t>(ch, 128u);
    const uint32_t ns_r = (uint32_t)(minrows / stride), ns = ns_r * (uint32_t)world;
    if (ns >= 4096 && !getenv("XKNN_NO_PILOT")) {
      const uint32_t nspad = (ns + 255) / 256 * 256;
      __half* s16 = nullptr;
      G_CUDA(mem.get(&s16, (uint64_t)nspad * 512));
      if (world == 1) {
        k_sample_rows<<<grid_for((uint64_t)nspad * 64, 256), 256, 0, s>>>(own16, stride, ns,
                                                                           nspad, s16);
      } else {
        k_sample_rows<<<grid_for((uint64_t)ns_r * 64, 256), 256, 0, s>>>(
            own16, stride, ns_r, ns_r, s16 + (uint64_t)rank * ns_r * 512);
        G_CUDA(cudaGetLastError());
        G_NCCL(ncclAllGather(s16 + (uint64_t)rank * ns_r * 512, s16, (size_t)ns_r * 512,
                             ncclFloat16, comm, s));
        if (nspad > ns)
          G_CUDA(cudaMemsetAsync(s16 + (uint64_t)ns * 512, 0, (size_t)(nspad - ns) * 1024, s));
      }
      G_CUDA(cudaGetLastError());
      // sample ids lie above every class id: the row itself is not masked (its score only
      // lowers the seed by one rank)
      G_CUDA(launch_graph_candidates(own16, n, row_base, s16, ns, 0xffffffffu - ns - n, list,
                                     lcnt, lcut, 32, kc, cand, ccnt, ctau, pilot_ch, s));
      k_seed_cut<<<grid_for((uint64_t)n * 32, 256), 256, 0, s>>>(list, lcnt, lcut, n, kc, jseed);
      G_CUDA(cudaGetLastError());
      mem.release(s16);
    }
  }
  if (timing) G_CUDA(cudaEventRecord(tev[5], s));
  // diagnostic (XKNN_GRAPH_SCAN_ONLY=<cut>): every row's cut starts at <cut>; the build stops
  // after the candidate pass (scan cost without inserts for a cut above every score)
  const char* scan_only = n >= 100000 ? getenv("XKNN_GRAPH_SCAN_ONLY") : nullptr;
  if (scan_only) {
    std::vector<float> hc(n, (float)atof(scan_only));
    G_CUDA(cudaMemcpyAsync(lcut, hc.data(), (size_t)n * 4, cudaMemcpyHostToDevice, s));
    G_CUDA(cudaStreamSynchronize(s));
  }
  const __half* held = own16;
  for (int h = 0; h < world; ++h) {
    const int o = (rank - h + world) % world;
    uint64_t cb, ce;
    shard_range_of(n_total, world, o, &cb, &ce);
    cudaEvent_t ev_recv = nullptr;
    if (h + 1 < world) {
      // pass the held block on (rank -> rank+1) while it is scored here; the receive buffer
      // was last read by the previous hop's GEMM
      cudaEvent_t ev_ready;
      G_CUDA(new_event(&ev_ready));
      G_CUDA(cudaEventRecord(ev_ready, s));
      G_CUDA(cudaStreamWaitEvent(cs, ev_ready, 0));
      const int po = (prev - h + world) % world;  // origin of the block prev holds at hop h
      uint64_t pb, pe;
      shard_range_of(n_total, world, po, &pb, &pe);
      G_NCCL(ncclGroupStart());
      G_NCCL(ncclSend(held, (ce - cb) * 512, ncclFloat16, next, comm, cs));
      G_NCCL(ncclRecv(buf16[h % 2], (pe - pb) * 512, ncclFloat16, prev, comm, cs));
      G_NCCL(ncclGroupEnd());
      G_CUDA(new_event(&ev_recv));
      G_CUDA(cudaEventRecord(ev_recv, cs));
    }
    G_CUDA(launch_graph_candidates(own16, n, row_base, held, (uint32_t)(ce - cb), (uint32_t)cb,
                                   list, lcnt, lcut, kp, kc, cand, ccnt, ctau, ch, s));
    if (h + 1 < world) {
      G_CUDA(cudaStreamWaitEvent(s, ev_recv, 0));
      held = buf16[h % 2];
      if (stats) ++stats->transfer_steps;
    }
  }
  if (getenv("XKNN_GRAPH_DEBUG")) {
    G_CUDA(cudaStreamSynchronize(s));
    std::vector<uint32_t> hc(n);
    std::vector<float> ht(n);
    cudaMemcpy(hc.data(), lcnt, (size_t)n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ht.data(), lcut, (size_t)n * 4, cudaMemcpyDeviceToHost);
    for (uint32_t j : {0u, 1u, n / 2, n - 1})
      fprintf(stderr, "rank %d row %u: list %u cut %g\n", rank, row_base + j, hc[j], ht[j]);
  }
  mem.release(cand);
  mem.release(own16);
  mem.release(buf16[0]);
  mem.release(buf16[1]);

  // ---- 2. certificate + window ----
  if (timing) G_CUDA(cudaEventRecord(tev[1], s));
  if (scan_only) {
    G_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, tev[5], tev[1]);
    fprintf(stderr, "[xknn graph] scan only (cut %s): candidates %.2f ms\n", scan_only, ms);
    return fail_msg(XKNN_ERR_UNSUPPORTED, "XKNN_GRAPH_SCAN_ONLY diagnostic");
  }
  G_CUDA(mem.get(&flag, n));
  G_CUDA(mem.get(&unc, (uint64_t)n + 1));
  G_CUDA(cudaMemsetAsync(unc, 0, 4, s));
  k_window<<<grid_for((uint64_t)n * 32, 256), 256, 0, s>>>(list, lcnt, lcut, n, kc, need, flag, unc,
                                                           unc + 1);
  G_CUDA(cudaGetLastError());
  uint32_t nu = 0;
  G_CUDA(cudaMemcpyAsync(&nu, unc, 4, cudaMemcpyDeviceToHost, s));
  G_CUDA(cudaStreamSynchronize(s));
  if (stats) stats->uncertified_rows = nu;

  // ---- 3. exact ring (fp32) ----
  if (timing) G_CUDA(cudaEventRecord(tev[2], s));
  G_CUDA(mem.get(&ex, (uint64_t)n * kc));
  float* buf32[2] = {nullptr, nullptr};
  if (world > 1) {
    G_CUDA(mem.get(&buf32[0], maxrows * 512));
    G_CUDA(mem.get(&buf32[1], maxrows * 512));
  }
  const uint32_t ulen = (uint32_t)world * need;
  float2* ubuf = nullptr;
  if (nu) G_CUDA(mem.get(&ubuf, (uint64_t)nu * ulen));
  const float* held32 = wn;
  for (int h = 0; h < world; ++h) {
    const int o = (rank - h + world) % world;
    uint64_t cb, ce;
    shard_range_of(n_total, world, o, &cb, &ce);
    const uint32_t nc = (uint32_t)(ce - cb);
    cudaEvent_t ev_recv = nullptr;
    if (h + 1 < world) {
      cudaEvent_t ev_ready;
      G_CUDA(new_event(&ev_ready));
      G_CUDA(cudaEventRecord(ev_ready, s));
      G_CUDA(cudaStreamWaitEvent(cs, ev_ready, 0));
      const int po = (prev - h + world) % world;
      uint64_t pb, pe;
      shard_range_of(n_total, world, po, &pb, &pe);
      G_NCCL(ncclGroupStart());
      G_NCCL(ncclSend(held32, (ce - cb) * 512, ncclFloat, next, comm, cs));
      G_NCCL(ncclRecv(buf32[h % 2], (pe - pb) * 512, ncclFloat, prev, comm, cs));
      G_NCCL(ncclGroupEnd());
      G_CUDA(new_event(&ev_recv));
      G_CUDA(cudaEventRecord(ev_recv, cs));
    }
    G_CUDA(cudaFuncSetAttribute(k_rescore, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kRescoreSmem));
    k_rescore<<<grid_for((uint64_t)n * 32, 256), 256, kRescoreSmem, s>>>(wn, n, 512, list, lcnt, flag, kc,
                                                              held32, (uint32_t)cb, nc, ex);
    G_CUDA(cudaGetLastError());
    // rows without a certificate: exact top-`need` against the whole block, batched
    G_CUDA(exact_topk(wn, unc + 1, nu, row_base, held32, nc, 512, (uint32_t)cb, need,
                      ubuf + (uint64_t)h * need, ulen, mem, s));
    if (h + 1 < world) {
      G_CUDA(cudaStreamWaitEvent(s, ev_recv, 0));
      held32 = buf32[h % 2];
    }
  }

  // ---- 4. finalize ----
  if (timing) G_CUDA(cudaEventRecord(tev[3], s));
  {
    uint32_t cap = 1;
    while (cap < std::max(kc, nu ? ulen : 1u)) cap <<= 1;
    const uint32_t warps = 4;
    const size_t smem = (size_t)warps * cap * 8;
    if (smem > 48 * 1024)
      G_CUDA(cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    k_finalize<<<grid_for((uint64_t)n * 32, warps * 32, 148u * 32u), warps * 32, smem, s>>>(
        n, row_base, k, kc, cap, list, lcnt, ex, flag, ubuf, ulen, out);
    G_CUDA(cudaGetLastError());
  }
  if (timing) G_CUDA(cudaEventRecord(tev[4], s));
  G_CUDA(cudaStreamSynchronize(s));
  if (cs) G_CUDA(cudaStreamSynchronize(cs));
  if (timing) {
    float ms[5];
    for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&ms[i], tev[i], tev[i + 1]);
    cudaEventElapsedTime(&ms[4], tev[0], tev[5]);
    fprintf(stderr,
            "[xknn graph] rank %d rows %u k %u k' %u: candidates %.2f ms (pilot %.2f), window %.2f "
            "ms, exact ring %.2f ms, finalize %.2f ms, uncertified %u\n",
            rank, n, k, kp, ms[0], ms[4], ms[1], ms[2], ms[3], nu);
  }
#undef G_CUDA
#undef G_NCCL
  return XKNN_OK;
}

// classify_retrieval on one shard: for each normalized query (qn, nq x 512)
// the exactly best class among the normalized rows wn (nw x 512, global ids col_base..) --
// argmax of the reference-order fp32 cosine, ties to the lower id -- by the graph build's
// scheme with one neighbour and no self: fp16 tensor-core candidates (up to 32 per query above
// a cut), the certificate A_1 > T + 2 eps, exact re-scores of the window, exact scans for the
// uncertified.  best_score / best_id: nq each, device.
xknn_status_t retrieval_top1_local(const float* qn, uint32_t nq, const float* wn, uint32_t nw,
                                   uint32_t col_base, uint32_t d, cudaStream_t s,
                                   float* best_score, uint32_t* best_id, uint64_t* uncertified) {
  cudaError_t e = cudaSuccess;
#define G_CUDA(x)                                                         \
  do {                                                                    \
    e = (x);                                                              \
    if (e != cudaSuccess) return fail_msg(XKNN_ERR_CUDA, cudaGetErrorString(e)); \
  } while (0)
  if ((uint64_t)col_base + nw + nq >= 0xffffffffull)
    return fail_msg(XKNN_ERR_UNSUPPORTED, "classify: class ids + queries must fit u32");
  const uint32_t kp = 32, kc = 64, ch = 64;
  Dev mem(s);
  float2* list = nullptr;
  uint32_t *lcnt = nullptr, *flag = nullptr, *unc = nullptr;
  float *lcut = nullptr, *ex = nullptr;
  G_CUDA(mem.get(&list, (uint64_t)nq * kc));
  G_CUDA(mem.get(&lcnt, nq));
  G_CUDA(mem.get(&lcut, nq));
  G_CUDA(mem.get(&flag, nq));
  G_CUDA(mem.get(&unc, (uint64_t)nq + 1));
  G_CUDA(mem.get(&ex, (uint64_t)nq * kc));
  G_CUDA(cudaMemsetAsync(unc, 0, 4, s));
  uint32_t nu = 0;
  if (d == 512) {
    const uint64_t qpad = (nq + 255) / 256 * 256, wpad = ((uint64_t)nw + 255) / 256 * 256;
    __half *q16 = nullptr, *w16 = nullptr;
    float2* cand = nullptr;
    uint32_t* ccnt = nullptr;
    float* ctau = nullptr;
    G_CUDA(mem.get(&q16, qpad * 512));
    G_CUDA(mem.get(&w16, wpad * 512));
    G_CUDA(mem.get(&cand, (uint64_t)kNumSMs / 2 * 256 * 2 * ch));
    G_CUDA(mem.get(&ccnt, (uint64_t)kNumSMs / 2 * 256 * 2));
    G_CUDA(mem.get(&ctau, (uint64_t)kNumSMs / 2 * 256 * 2));
    k_to_f16<<<grid_for(qpad * 256, 256), 256, 0, s>>>(qn, nq, qpad, 512, q16);
    k_to_f16<<<grid_for(wpad * 256, 256), 256, 0, s>>>(wn, nw, wpad, 512, w16);
    k_list_init<<<grid_for(nq, 256), 256, 0, s>>>(lcnt, lcut, nq);
    G_CUDA(cudaGetLastError());
    // queries are not classes: their "self" ids lie above every class id
    G_CUDA(launch_graph_candidates(q16, nq, 0xffffffffu - nq, w16, nw, col_base, list, lcnt, lcut,
                                   kp, kc, cand, ccnt, ctau, ch, s));
    k_window<<<grid_for((uint64_t)nq * 32, 256), 256, 0, s>>>(list, lcnt, lcut, nq, kc, 1, flag,
                                                              unc, unc + 1);
    G_CUDA(cudaGetLastError());
    G_CUDA(cudaMemcpyAsync(&nu, unc, 4, cudaMemcpyDeviceToHost, s));
    G_CUDA(cudaStreamSynchronize(s));
    G_CUDA(cudaFuncSetAttribute(k_rescore, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kRescoreSmem));
    k_rescore<<<grid_for((uint64_t)nq * 32, 256), 256, kRescoreSmem, s>>>(qn, nq, 512, list, lcnt, flag, kc,
                                                               wn, col_base, nw, ex);
    G_CUDA(cudaGetLastError());
  } else {  // exact scans for every query
    nu = nq;
    std::vector<uint32_t> ids(nq);
    for (uint32_t j = 0; j < nq; ++j) ids[j] = j;
    std::vector<uint32_t> fl(nq);
    for (uint32_t j = 0; j < nq; ++j) fl[j] = j + 1;
    G_CUDA(cudaMemcpyAsync(unc + 1, ids.data(), (size_t)nq * 4, cudaMemcpyHostToDevice, s));
    G_CUDA(cudaMemcpyAsync(flag, fl.data(), (size_t)nq * 4, cudaMemcpyHostToDevice, s));
    G_CUDA(cudaStreamSynchronize(s));
  }
  float2* ubuf = nullptr;
  if (nu) {  // queries without a certificate: exact best against every class row, batched
    G_CUDA(mem.get(&ubuf, nu));
    G_CUDA(exact_topk(qn, unc + 1, nu, 0xffffffffu, wn, nw, d, col_base, 1, ubuf, 1, mem, s));
  }
  k_top1<<<grid_for((uint64_t)nq * 32, 256), 256, 0, s>>>(nq, kc, list, lcnt, ex, flag, ubuf,
                                                          best_score, best_id);
  G_CUDA(cudaGetLastError());
  G_CUDA(cudaStreamSynchronize(s));
  if (uncertified) *uncertified = nu;
#undef G_CUDA
  return XKNN_OK;
}

}  // namespace xknn

extern "C" xknn_status_t xknn_graph_bruteforce(const float* w_norm_dev, uint64_t num_classes,
                                               uint64_t dim, uint32_t k, uint32_t kprime,
                                               uint32_t* out_dev, void* stream,
                                               uint64_t* uncertified_rows) {
  xknn::GraphBuildStats st{};
  xknn_status_t r = xknn::graph_build(w_norm_dev, num_classes, dim, k, kprime, 0, 1, nullptr,
                                      static_cast<cudaStream_t>(stream), out_dev, &st);
  if (uncertified_rows) *uncertified_rows = st.uncertified_rows;
  return r;
}

extern "C" xknn_status_t xknn_graph_release_cache(void) {
  int dev = 0;
  cudaMemPool_t pool = nullptr;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetDefaultMemPool(&pool, dev);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemPoolTrimTo(pool, 0);
  return e == cudaSuccess ? XKNN_OK : xknn::fail_msg(XKNN_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" xknn_status_t xknn_graph_ring(const float* w_norm_local_dev, uint64_t num_classes,
                                         uint64_t dim, uint32_t k, uint32_t kprime, int rank,
                                         int world, void* comm, void* stream,
                                         uint32_t* out_rows_dev, uint64_t* uncertified_rows,
                                         uint64_t* transfer_steps) {
  if (kprime < k)
    return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "build_graph_ring: k' must be >= k");
  xknn::GraphBuildStats st{};
  xknn_status_t r = xknn::graph_build(w_norm_local_dev, num_classes, dim, k, kprime, rank, world,
                                      static_cast<ncclComm_t>(comm),
                                      static_cast<cudaStream_t>(stream), out_rows_dev, &st);
  if (uncertified_rows) *uncertified_rows = st.uncertified_rows;
  if (transfer_steps) *transfer_steps = st.transfer_steps;
  return r;
}
