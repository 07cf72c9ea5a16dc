// rowops.cu -- HBM-bound row kernels shared by both precisions: feature normalize, active-row
// gather + normalize, normalize-backward fused with the sparse momentum-SGD update, and the
// feature normalize-backward.  One warp per 512-float row, 16-byte vector loads/stores.
//
// Arithmetic follows the reference op-for-op in fp32 (no FMA contraction: __fmul_rn/__fadd_rn)
// with fp64 row reductions:
//   l2_normalize_rows_cached  matrix.cpp:12-29     norm = float(sqrt(sum double(x^2)))
//   l2_normalize_backward     matrix.cpp:31-48     (g - float(sum double(g*x_hat)) * x_hat) / |x|
//   inline W backward         parallel.cpp:653-666
//   SgdMomentum::step_rows    fccs.cpp:74-89       v = (mu*v + g) + wd*w ; w -= lr*v
#include "kernels.cuh"

namespace xknn {

namespace {

template <typename T>
__device__ __forceinline__ T warp_allsum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(XKNN_FULL_MASK, v, o);
  return v;
}

__device__ __forceinline__ void store_bf16x4(__nv_bfloat16* dst, float a, float b, float c,
                                             float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b);
  __nv_bfloat162 hi = __floats2bfloat162_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(dst) = u;
}

// D is a multiple of 128 (checked at create); each lane owns D/128 float4 chunks.
// SEQ: the fp64 sum of squares in ascending column order, as matrix.cpp:18-21 (FP32_EXACT, whose
// logits are bit-identical to the reference's); otherwise lane-strided partials + a butterfly
// (the norm may differ from the reference's in the last bit for ~2^-28 of rows).
template <int DV, bool SEQ = false>  // DV = D/128 float4 per lane
__global__ void k_normalize_rows(const float* __restrict__ in, uint64_t rows, uint32_t d,
                                 const uint32_t* __restrict__ row_ids, const unsigned int* count,
                                 uint64_t id_base, float* __restrict__ out32,
                                 __nv_bfloat16* __restrict__ out16, float* __restrict__ norms,
                                 unsigned long long* err, float* __restrict__ out_lo,
                                 __nv_bfloat16* __restrict__ out16_lo,
                                 __nv_bfloat16* __restrict__ out_d) {
  griddep_wait();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nrows = count ? *count : rows;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < nrows;
       r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint64_t src_row = row_ids ? (uint64_t)row_ids[r] - id_base : r;
    const float4* src = reinterpret_cast<const float4*>(in + src_row * d);
    float4 v[DV];
    double sq = 0.0;
#pragma unroll
    for (int c = 0; c < DV; ++c) {
      v[c] = src[lane + 32 * c];
      if (!SEQ) {
        sq += (double)v[c].x * v[c].x;
        sq += (double)v[c].y * v[c].y;
        sq += (double)v[c].z * v[c].z;
        sq += (double)v[c].w * v[c].w;
      }
    }
    if (SEQ) {  // every lane runs the same column-order chain on broadcast values
#pragma unroll
      for (int c = 0; c < DV; ++c)
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
          const float a = __shfl_sync(XKNN_FULL_MASK, v[c].x, j);
          const float b = __shfl_sync(XKNN_FULL_MASK, v[c].y, j);
          const float e = __shfl_sync(XKNN_FULL_MASK, v[c].z, j);
          const float f = __shfl_sync(XKNN_FULL_MASK, v[c].w, j);
          sq += (double)a * a;
          sq += (double)b * b;
          sq += (double)e * e;
          sq += (double)f * f;
        }
    } else {
      sq = warp_allsum(sq);
    }
    const float norm = (float)sqrt(sq);
    if (norm < 1e-12f) {
      if (lane == 0) raise_error(err, XKNN_ERR_ZERO_NORM_ROW, r);
      continue;
    }
    if (lane == 0 && norms) norms[r] = norm;
    const float inv = 1.0f / norm;
#pragma unroll
    for (int c = 0; c < DV; ++c) {
      float4 o;
      o.x = __fmul_rn(v[c].x, inv);
      o.y = __fmul_rn(v[c].y, inv);
      o.z = __fmul_rn(v[c].z, inv);
      o.w = __fmul_rn(v[c].w, inv);
      const uint64_t col = (uint64_t)(lane + 32 * c) * 4;
      if (out_lo || out_d) {  // tf32 operand split: out32 = tf32(o) (round to nearest), and
                              // o - it in fp32 (3xTF32, out_lo) or bf16 (mixed GEMM-F, out_d)
        const float4 hi = make_float4(tf32_rna(o.x), tf32_rna(o.y), tf32_rna(o.z), tf32_rna(o.w));
        *reinterpret_cast<float4*>(out32 + r * d + col) = hi;
        const float4 lo = make_float4(o.x - hi.x, o.y - hi.y, o.z - hi.z, o.w - hi.w);
        if (out_lo) *reinterpret_cast<float4*>(out_lo + r * d + col) = lo;
        if (out_d) store_bf16x4(out_d + r * d + col, lo.x, lo.y, lo.z, lo.w);
      } else if (out32) {
        *reinterpret_cast<float4*>(out32 + r * d + col) = o;
      }
      if (out16_lo) {  // bf16 planes (bf16x3 GEMM operand): out16 = bf16(o), out16_lo = bf16(o - it)
        const __nv_bfloat162 h0 = __floats2bfloat162_rn(o.x, o.y), h1 = __floats2bfloat162_rn(o.z, o.w);
        const float2 f0 = __bfloat1622float2(h0), f1 = __bfloat1622float2(h1);
        uint2 u;
        u.x = *reinterpret_cast<const uint32_t*>(&h0);
        u.y = *reinterpret_cast<const uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(out16 + r * d + col) = u;
        store_bf16x4(out16_lo + r * d + col, o.x - f0.x, o.y - f0.y, o.z - f1.x, o.w - f1.y);
      } else if (out16) {
        store_bf16x4(out16 + r * d + col, o.x, o.y, o.z, o.w);
      }
    }
  }
}

// Normalize-backward of each active row through its cached norm, then SgdMomentum::step_rows
// on (W, V).  g rows are compact (row t <-> active[t]), minus the one-hot correction of
// LabelFix.  Parameters are not touched if any error was raised earlier in the step (the
// reference throws before touching parameters); the label lists are cleared either way.
__device__ __forceinline__ float4 load_g4(const float* __restrict__ G, uint64_t i) {
  return reinterpret_cast<const float4*>(G)[i];
}
__device__ __forceinline__ float4 load_g4(const __nv_bfloat16* __restrict__ G, uint64_t i) {
  const uint2 u = reinterpret_cast<const uint2*>(G)[i];
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                     __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
}

#ifndef XKNN_UPD_MINB
#define XKNN_UPD_MINB 2
#endif
template <int DV, typename GT = float, bool SPLIT = false>
__global__ void __launch_bounds__(256, XKNN_UPD_MINB)
    k_update_rows(float* __restrict__ W, float* __restrict__ V,
                              const GT* __restrict__ G, const uint32_t* __restrict__ active,
                              const unsigned int* count, uint64_t begin, uint32_t d,
                              const float* __restrict__ wnorm, const float* __restrict__ lr_dev,
                              float mu, float wd, const unsigned long long* err, LabelFix lf) {
  griddep_wait();
  const bool dead = *err != 0;
  if (dead && !lf.head) return;
  const float lr = *lr_dev;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nrows = *count;
  for (uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; t < nrows;
       t += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    // the batch rows labelled with this class (lists are almost always empty or 1 long); the
    // list head is cleared after the row's last access (no load waits behind that store)
    const int32_t lh = lf.head ? lf.head[t] : -1;
    if (dead) {
      __syncwarp();
      if (lane == 0 && lh >= 0) lf.head[t] = -1;
      continue;
    }
    const uint64_t row = (uint64_t)active[t] - begin;
    float4* wp = reinterpret_cast<float4*>(W + row * d);
    float4* vp = reinterpret_cast<float4*>(V + row * d);
    const uint64_t g0 = t * d / 4;
    const float norm = wnorm[t];
    const float inv = 1.0f / norm;
    float4 w[DV], g[DV], nh[DV], vel[DV];
    double dot = 0.0;
    // every load of the row in flight before the first use (W, G, V: 3 x 2 KiB per warp)
#pragma unroll
    // a row of a split GEMM-dW tail unit: the sum of its fp32 K-partials, in part order
    const uint32_t unit = (uint32_t)(t / 256);
    bool split = false;
    DwSplit sp{0, 1};
    if (SPLIT) {
      sp = dw_split((uint32_t)((nrows + 255) / 256), lf.npairs);
      split = unit >= sp.full;
    }
#pragma unroll
    for (int c = 0; c < DV; ++c) {
      w[c] = wp[lane + 32 * c];
      if (!split) g[c] = load_g4(G, g0 + lane + 32 * c);
      vel[c] = vp[lane + 32 * c];
    }
    if (split) {
      const uint64_t slot0 = (uint64_t)(unit - sp.full) * sp.s;
      const float4* pp = reinterpret_cast<const float4*>(lf.dw_part) +
                         ((slot0 * 256 + t % 256) * (uint64_t)d) / 4;
#pragma unroll
      for (int c = 0; c < DV; ++c) g[c] = pp[lane + 32 * c];
      for (uint32_t q = 1; q < sp.s; ++q) {
        const float4* pq = pp + (uint64_t)q * 256 * d / 4;
#pragma unroll
        for (int c = 0; c < DV; ++c) {
          const float4 y = pq[lane + 32 * c];
          g[c].x = __fadd_rn(g[c].x, y.x);
          g[c].y = __fadd_rn(g[c].y, y.y);
          g[c].z = __fadd_rn(g[c].z, y.z);
          g[c].w = __fadd_rn(g[c].w, y.w);
        }
      }
    }
    if (lh >= 0) {
      float4 xs[DV];
#pragma unroll
      for (int c = 0; c < DV; ++c) xs[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      int32_t cur = -1;
      for (;;) {  // next larger batch row of the list (every lane walks it: broadcast loads)
        int32_t best = INT32_MAX;
        for (int32_t b = lh; b >= 0; b = lf.next[b])
          if (b > cur && b < best) best = b;
        if (best == INT32_MAX) break;
        cur = best;
        const float xi = 1.0f / lf.xnorm[cur];
        const float4* xp = reinterpret_cast<const float4*>(lf.X + (uint64_t)cur * d);
#pragma unroll
        for (int c = 0; c < DV; ++c) {
          const float4 x = xp[lane + 32 * c];
          xs[c].x = __fadd_rn(xs[c].x, __fmul_rn(x.x, xi));
          xs[c].y = __fadd_rn(xs[c].y, __fmul_rn(x.y, xi));
          xs[c].z = __fadd_rn(xs[c].z, __fmul_rn(x.z, xi));
          xs[c].w = __fadd_rn(xs[c].w, __fmul_rn(x.w, xi));
        }
      }
#pragma unroll
      for (int c = 0; c < DV; ++c) {
        g[c].x = __fsub_rn(g[c].x, __fmul_rn(lf.sb, xs[c].x));
        g[c].y = __fsub_rn(g[c].y, __fmul_rn(lf.sb, xs[c].y));
        g[c].z = __fsub_rn(g[c].z, __fmul_rn(lf.sb, xs[c].z));
        g[c].w = __fsub_rn(g[c].w, __fmul_rn(lf.sb, xs[c].w));
      }
    }
#pragma unroll
    for (int c = 0; c < DV; ++c) {
      nh[c].x = __fmul_rn(w[c].x, inv);
      nh[c].y = __fmul_rn(w[c].y, inv);
      nh[c].z = __fmul_rn(w[c].z, inv);
      nh[c].w = __fmul_rn(w[c].w, inv);
      dot += (double)g[c].x * nh[c].x;
      dot += (double)g[c].y * nh[c].y;
      dot += (double)g[c].z * nh[c].z;
      dot += (double)g[c].w * nh[c].w;
    }
    dot = warp_allsum(dot);
    const float dd = (float)dot;
    const float inv2 = 1.0f / norm;
#pragma unroll
    for (int c = 0; c < DV; ++c) {
      float4 v = vel[c];
      float gr, vv;
#define XKNN_UPD(comp)                                                                  \
  gr = __fmul_rn(__fsub_rn(g[c].comp, __fmul_rn(dd, nh[c].comp)), inv2);               \
  vv = __fadd_rn(__fadd_rn(__fmul_rn(mu, v.comp), gr), __fmul_rn(wd, w[c].comp));      \
  v.comp = vv;                                                                          \
  w[c].comp = __fsub_rn(w[c].comp, __fmul_rn(lr, vv));
      XKNN_UPD(x) XKNN_UPD(y) XKNN_UPD(z) XKNN_UPD(w)
#undef XKNN_UPD
      vp[lane + 32 * c] = v;
      wp[lane + 32 * c] = w[c];
    }
    if (lh >= 0) {
      __syncwarp();
      if (lane == 0) lf.head[t] = -1;
    }
  }
}

// gfeat = l2_normalize_backward(x_hat, norms, g) for this rank's rows; x_hat recomputed from the
// raw features exactly as the forward did.
template <int DV>
// micros > 1: row r of the rank's slice belongs to micro-batch c of the balanced split
// (parallel.cpp:514-523), whose softmax gradient carries 1/m_c instead of 1/m; the gradient the
// reference hands to mlp_backward for that row is this one times m/m_c = rows/rows_c.
__global__ void k_feature_backward(const float* __restrict__ X, const float* __restrict__ xnorm,
                                   const float* __restrict__ G, uint64_t rows, uint32_t d,
                                   float* __restrict__ out, uint32_t micros) {
  griddep_wait();
  griddep_launch();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t mb = micros > rows ? rows : (micros ? micros : 1);
  const uint64_t mbase = rows / mb, mrem = rows % mb;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint64_t rows_c = r < mrem * (mbase + 1) ? mbase + 1 : mbase;
    const float mf = mb > 1 ? (float)((double)rows / (double)rows_c) : 1.0f;
    const float norm = xnorm[r];
    const float inv = 1.0f / norm;
    const float4* xp = reinterpret_cast<const float4*>(X + r * d);
    const float4* gp = reinterpret_cast<const float4*>(G + r * d);
    float4 nh[DV], g[DV];
    double dot = 0.0;
#pragma unroll
    for (int c = 0; c < DV; ++c) {
      const float4 x = xp[lane + 32 * c];
      g[c] = gp[lane + 32 * c];
      if (mb > 1) {
        g[c].x = __fmul_rn(g[c].x, mf);
        g[c].y = __fmul_rn(g[c].y, mf);
        g[c].z = __fmul_rn(g[c].z, mf);
        g[c].w = __fmul_rn(g[c].w, mf);
      }
      nh[c].x = __fmul_rn(x.x, inv);
      nh[c].y = __fmul_rn(x.y, inv);
      nh[c].z = __fmul_rn(x.z, inv);
      nh[c].w = __fmul_rn(x.w, inv);
      dot += (double)g[c].x * nh[c].x;
      dot += (double)g[c].y * nh[c].y;
      dot += (double)g[c].z * nh[c].z;
      dot += (double)g[c].w * nh[c].w;
    }
    dot = warp_allsum(dot);
    const float dd = (float)dot;
    const float inv2 = 1.0f / norm;
#pragma unroll
    for (int c = 0; c < DV; ++c) {
      float4 o;
      o.x = __fmul_rn(__fsub_rn(g[c].x, __fmul_rn(dd, nh[c].x)), inv2);
      o.y = __fmul_rn(__fsub_rn(g[c].y, __fmul_rn(dd, nh[c].y)), inv2);
      o.z = __fmul_rn(__fsub_rn(g[c].z, __fmul_rn(dd, nh[c].z)), inv2);
      o.w = __fmul_rn(__fsub_rn(g[c].w, __fmul_rn(dd, nh[c].w)), inv2);
      reinterpret_cast<float4*>(out + r * d)[lane + 32 * c] = o;
    }
  }
}

}  // namespace

#define XKNN_DISPATCH_D(d, KERNEL, GRID, BLOCK, STREAM, ...)                              \
  switch ((d) / 128) {                                                                    \
    case 1: launch_pdl(KERNEL<1>, GRID, BLOCK, 0, STREAM, __VA_ARGS__); break;                    \
    case 2: launch_pdl(KERNEL<2>, GRID, BLOCK, 0, STREAM, __VA_ARGS__); break;                    \
    case 4: launch_pdl(KERNEL<4>, GRID, BLOCK, 0, STREAM, __VA_ARGS__); break;                    \
    case 8: launch_pdl(KERNEL<8>, GRID, BLOCK, 0, STREAM, __VA_ARGS__); break;                    \
    default: return cudaErrorInvalidValue;                                                \
  }

cudaError_t launch_normalize_rows(const float* in, uint64_t rows, uint32_t d,
                                  const uint32_t* row_ids, const unsigned int* count,
                                  uint64_t id_base, float* out32, __nv_bfloat16* out16,
                                  float* norms, unsigned long long* err, cudaStream_t s,
                                  bool seq, float* out_lo, __nv_bfloat16* out16_lo,
                                  __nv_bfloat16* out_d) {
  const unsigned grid = grid_for(rows * 32, 256);
  if (seq) {
#define XKNN_SEQ_CASE(DV)                                                                      \
  case DV:                                                                                     \
    launch_pdl(k_normalize_rows<DV, true>, grid, 256, 0, s, in, rows, d, row_ids, count, id_base, \
               out32, out16, norms, err, out_lo, out16_lo, out_d);                             \
    break;
    switch (d / 128) {
      XKNN_SEQ_CASE(1) XKNN_SEQ_CASE(2) XKNN_SEQ_CASE(4) XKNN_SEQ_CASE(8)
      default: return cudaErrorInvalidValue;
    }
#undef XKNN_SEQ_CASE
    return cudaGetLastError();
  }
  XKNN_DISPATCH_D(d, k_normalize_rows, grid, 256, s, in, rows, d, row_ids, count, id_base, out32,
                  out16, norms, err, out_lo, out16_lo, out_d);
  return cudaGetLastError();
}

cudaError_t launch_update_rows(float* W, float* V, const float* G, const uint32_t* active,
                               const unsigned int* count, uint64_t max_rows, uint64_t begin,
                               uint32_t d, const float* wnorm, const float* lr, float mu, float wd,
                               const unsigned long long* err, cudaStream_t s, unsigned max_grid,
                               LabelFix lf) {
  const unsigned grid = grid_for(max_rows * 32, 256, max_grid);
  if (lf.dw_part) {  // rows of split GEMM-dW tail units arrive as K-partials (FP32 path, D = 512)
    if (d != 512) return cudaErrorInvalidValue;
    launch_pdl(k_update_rows<4, float, true>, grid, 256, 0, s, W, V, G, active, count, begin, d,
               wnorm, lr, mu, wd, err, lf);
    return cudaGetLastError();
  }
  XKNN_DISPATCH_D(d, k_update_rows, grid, 256, s, W, V, G, active, count, begin, d, wnorm, lr, mu,
                  wd, err, lf);
  return cudaGetLastError();
}

cudaError_t launch_update_rows_bf16(float* W, float* V, const __nv_bfloat16* G,
                                    const uint32_t* active, const unsigned int* count,
                                    uint64_t max_rows, uint64_t begin, uint32_t d,
                                    const float* wnorm, const float* lr, float mu, float wd,
                                    const unsigned long long* err, cudaStream_t s,
                                    LabelFix lf) {
  if (d != 512) return cudaErrorInvalidValue;
  const unsigned grid = grid_for(max_rows * 32, 256, 148u * 16u);
  launch_pdl(k_update_rows<4, __nv_bfloat16>, grid, 256, 0, s, W, V, G, active, count, begin, d, wnorm,
                                                       lr, mu, wd, err, lf);
  return cudaGetLastError();
}

cudaError_t launch_feature_backward(const float* X, const float* xnorm, const float* G,
                                    uint64_t rows, uint32_t d, float* out, cudaStream_t s,
                                    uint32_t micros) {
  const unsigned grid = grid_for(rows * 32, 256);
  XKNN_DISPATCH_D(d, k_feature_backward, grid, 256, s, X, xnorm, G, rows, d, out, micros);
  return cudaGetLastError();
}

}  // namespace xknn
