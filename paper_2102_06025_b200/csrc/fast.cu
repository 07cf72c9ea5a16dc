// fast.cu -- XKNN_PREC_BF16: the three fc GEMMs on 5th-gen tensor cores (tcgen05.mma,
// accumulators in TMEM, operands staged by TMA into 128B/64B-swizzled shared memory), with the
// softmax fused into the forward epilogue so logits never reach HBM.
//
// Forward (parallel.cpp:550-557, the logits GEMM + softmax statistics):
//   GEMM-F   S = X_hat * W_subᵀ   (M = 128 batch rows, N = 256 classes, K = D)
//            epilogue: P~ = exp(s*S - s) -> bf16 (B x M_w), per-tile row sums, label logit.
//            A fixed stabiliser c = s replaces the row max: |cosine| <= 1 bounds every logit
//            to [-s, s], so exp(s*S - s) lies in [e^-2s, 1] (fp32-safe for s <= 40).
// Backward, with r_b = 1 / (B * sum_b), G = r * P~ - onehot / B (= softmax - onehot over m,
// parallel.cpp:168-186):
//   GEMM-dW  dW  = P~ᵀ * (diag(s*r) X_hat)     (M = 128 classes, N = 512, K = B) -> bf16 rows
//   GEMM-dX  dX  = diag(s*r) * (P~ * W_sub)    (M = 128 batch, N = 512, K = M_w split) -> fp32
// The one-hot term is a sparse fp32 rank-B correction, never rounded to bf16: k_dx_reduce
// subtracts (s/B) * w_hat[y_b] from feature row b, and the row update subtracts
// (s/B) * sum{x_hat_b : y_b = class} from the class's dW row (label lists built by k_fixup).
// Warp roles (384 threads, one CTA per SM, persistent over tiles): warp 0 TMA producer,
// warp 1 MMA issuer (one thread), warp 2 TMEM allocator, warps 4-11 epilogue (TMEM -> regs).
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include "kernels.cuh"
#include "tc.cuh"

namespace xknn {

namespace {

enum Kind : int { kF = 0, kDX = 1, kDW = 2, kG = 3 };

__device__ __forceinline__ void epilogue_bar() {  // the 8 epilogue warps only
  asm volatile("bar.sync 1, 256;" ::: "memory");
}

struct GemmArgs {
  const SelState* st;
  uint32_t B, bpad, nbt, splits, dim;
  uint32_t dwsplit;  // GEMM-dW: split the tail units along K (dw_split) -- see Layer::run_fast_core
  float scale;
  const int32_t* label_col;
  __nv_bfloat16* Pt;
  uint64_t ldp;
  float* partial;
  float* labelterm;
  __nv_bfloat16* out16;  // GEMM-dW output rows (bf16, compact active order)
  // graph build (kG): own rows (A, global ids row_base..) against a held block of ncols
  // columns (B, global ids col_base..).  Per in-flight unit slot (pair * 256 + row): two
  // candidate regions [slot][half][ch] of (approx score, column id) with counts/cuts; per own
  // row: the persistent candidate list [row][kcap], its length and cut (every column not in
  // the list has approx score <= cut), merged at the end of each unit.
  float2* cand;
  uint32_t* cnt;
  float* tau;
  uint32_t ch, kprime, kcap, nrows, ncols;  // kcap: list capacity (row stride) >= kprime
  uint32_t row_base, col_base;
  uint32_t gchunk;  // kG: class tiles per column chunk (the L2-resident slice all pairs share)
  float2* list;
  uint32_t* lcnt;
  float* lcut;
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int KIND>
struct Cfg2;
template <>
struct Cfg2<kF> {  // P~ rows leave through one staging block per warp (plain stores)
  static constexpr uint32_t STAGES = 5, A_BYTES = 0, B_BYTES = 128 * 64 * 2;
  static constexpr uint32_t ARES_BYTES = 8 * 128 * 64 * 2;  // resident X_hat: 128 rows x 512
  static constexpr uint32_t NBUF = 2, ACC = 256, STG = 2048, NSTG = 1;
};
template <>
#ifndef XKNN_DX_KC
#define XKNN_DX_KC 64
#endif
struct Cfg2<kDX> {
  // KC classes of K per stage: A = this CTA's 128 batch rows x KC (P~, K-major, KC * 2 B rows),
  // B = KC rows x 4 atoms of 64 d (W_sub, MN-major) -- 64 fills the 128-B swizzle rows of A and
  // halves the stages (and TMA transactions / barrier round trips) per unit of work vs 32
  static constexpr uint32_t KC = XKNN_DX_KC;
  static constexpr uint32_t STAGES = KC == 64 ? 4 : 6, A_BYTES = 128 * KC * 2,
                            B_BYTES = 4 * 64 * KC * 2;
  static constexpr uint32_t ARES_BYTES = 0;
  static constexpr uint32_t NBUF = 1, ACC = 512, STG = 4096, NSTG = KC == 64 ? 1 : 2;
};
template <>
#ifndef XKNN_DW_KC
#define XKNN_DW_KC 64
#endif
struct Cfg2<kDW> {
  // KC batch rows of K per stage: A = 2 atoms of 64 classes x KC (P~ᵀ, MN-major), B = 4 atoms of
  // 64 d x KC (X_hat', MN-major)
  static constexpr uint32_t KC = XKNN_DW_KC;
  static constexpr uint32_t STAGES = KC == 64 ? 4 : 6, A_BYTES = 2 * 64 * KC * 2,
                            B_BYTES = 4 * 64 * KC * 2;
  static constexpr uint32_t ARES_BYTES = 0;
  // bf16 output: 2 KB per 32x32 chunk, NSTG chunks in flight per warp (the accumulator is
  // single-buffered, so the drain's store waits sit on the MMA's critical path)
  static constexpr uint32_t NBUF = 1, ACC = 512, STG = 2048, NSTG = KC == 64 ? 2 : 4;
};

template <>
struct Cfg2<kG> {
  static constexpr uint32_t STAGES = 6, A_BYTES = 0, B_BYTES = 128 * 64 * 2;
  static constexpr uint32_t ARES_BYTES = 8 * 128 * 64 * 2;
  static constexpr uint32_t NBUF = 2, ACC = 256, STG = 0, NSTG = 0;
};

template <int KIND>
constexpr uint32_t smem_bytes2() {
  using C = Cfg2<KIND>;
  return C::ARES_BYTES + C::STAGES * (C::A_BYTES + C::B_BYTES) + 8 * C::NSTG * C::STG + 1024 + 256 +
         (KIND == kG ? 1024 : 0);
}

struct Unit2 {
  uint32_t row0;   // F/dX: first batch row of the pair; dW: first class of the pair
  uint32_t t0, t1; // F: class-tile range; dX: K-chunk range; dW: K-stage range (batch rows)
  uint32_t id;     // dX: partial slot; dW: partial slot of a split tail unit
  bool valid;
  bool part;       // dW: a K-partial of a tail unit (fp32 partial rows, dw_split)
};

// Work units of one CTA pair.  With MCP = 2 the two pairs of a 4-CTA cluster take sibling
// units in lockstep -- different 256-row A tiles (batch tiles / query blocks), the same B stream
// -- and every B tile is fetched once per cluster and multicast to both pairs.
template <int KIND, int MCP>
__device__ __forceinline__ uint32_t num_units2(const GemmArgs& a, uint32_t mw) {
  if (KIND == kDW) {
    const uint32_t units = (mw + 255) / 256;
    const DwSplit sp = a.dwsplit ? dw_split(units, gridDim.x / (2 * MCP)) : DwSplit{units, 1};
    return sp.full + (units - sp.full) * sp.s;
  }
  if (KIND == kG) {  // chunk-major: every pair's row blocks against chunk 0, then chunk 1, ...
    const uint32_t npairs = gridDim.x / (2 * MCP);
    const uint32_t nrb = (a.nrows + 256 * MCP - 1) / (256 * MCP);
    const uint32_t nchunk = ((a.ncols + 255) / 256 + a.gchunk - 1) / a.gchunk;
    return nchunk * ((nrb + npairs - 1) / npairs) * npairs;
  }
  return a.nbt / MCP * a.splits;  // nbt = batch pair-tiles (256 rows), splits = ranges per tile
}


template <int KIND, int MCP>
__device__ __forceinline__ Unit2 unit2_of(const GemmArgs& a, uint32_t mw, uint32_t u,
                                          uint32_t pc) {
  Unit2 x{};
  x.id = u;
  if (KIND == kDW) {
    const uint32_t nk = a.bpad / Cfg2<kDW>::KC;
    const uint32_t units = (mw + 255) / 256;
    const DwSplit sp = a.dwsplit ? dw_split(units, gridDim.x / (2 * MCP)) : DwSplit{units, 1};
    x.valid = true;
    if (u < sp.full) {
      x.row0 = u * 256;
      x.t0 = 0;
      x.t1 = nk;
      return x;
    }
    const uint32_t v = u - sp.full, tt = v / sp.s, p = v % sp.s;
    x.row0 = (sp.full + tt) * 256;
    x.t0 = p * nk / sp.s;
    x.t1 = (p + 1) * nk / sp.s;
    x.id = v;  // = tt * s + p
    x.part = true;
    return x;
  }
  if (KIND == kG) {
    // one 256-row query block against one column chunk.  A pair owns the row blocks
    // rb = pair (mod npairs) and visits them chunk by chunk, so (i) a row's list is only ever
    // merged by one pair, in chunk order, and (ii) all pairs stream the same chunk at about the
    // same time: it is read from HBM once and served from L2 to every pair
    const uint32_t npairs = gridDim.x / (2 * MCP);
    const uint32_t nrb = (a.nrows + 256 * MCP - 1) / (256 * MCP);
    const uint32_t nrbp = (nrb + npairs - 1) / npairs;
    const uint32_t j = u / npairs, rb = (j % nrbp) * npairs + u % npairs;
    const uint32_t nt = (a.ncols + 255) / 256;
    x.row0 = (rb * MCP + pc) * 256;
    x.t0 = (j / nrbp) * a.gchunk;
    x.t1 = min(nt, x.t0 + a.gchunk);
    x.valid = rb < nrb && x.t1 > x.t0;
    return x;
  }
  const uint32_t nbc = a.nbt / MCP;
  const uint32_t bp = (u % nbc) * MCP + pc, r = u / nbc;
  x.id = bp + r * a.nbt;  // the pair-tile unit index (dX partial slots)
  const uint32_t nt = KIND == kF ? (mw + 255) / 256 : (mw + Cfg2<kDX>::KC - 1) / Cfg2<kDX>::KC;
  x.row0 = bp * 256;
  x.t0 = (uint32_t)((uint64_t)r * nt / a.splits);
  x.t1 = (uint32_t)((uint64_t)(r + 1) * nt / a.splits);
  x.valid = KIND == kDX || x.t1 > x.t0;  // dX units always write their (maybe zero) partial
  return x;
}

// swizzled staging of one thread's 32-element row chunk: fp32 (SW128, 128-B rows) or bf16
// (SW64, 64-B rows), matching the store tensor map
__device__ __forceinline__ void stage_f32(uint8_t* buf, uint32_t r, const float (&v)[32]) {
#pragma unroll
  for (uint32_t c = 0; c < 8; ++c) {
    float4* d = reinterpret_cast<float4*>(buf + r * 128 + ((c ^ (r & 7)) * 16));
    *d = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
}
__device__ __forceinline__ void stage_bf16(uint8_t* buf, uint32_t r, const uint32_t (&pk)[16]) {
#pragma unroll
  for (uint32_t c = 0; c < 4; ++c) {
    uint4* d = reinterpret_cast<uint4*>(buf + r * 64 + ((c ^ ((r >> 1) & 3)) * 16));
    *d = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
  }
}

// 32 rows x 32 bf16 of a 64-B-swizzled staging block (stage_bf16) to global rows `ld` elements
// apart: lane l writes row 8i + l/4, 16-B column unit l%4 -- eight 64-B row segments per
// instruction instead of 32 scattered ones, no async-proxy round trip.  Caller: __syncwarp()
// after staging; the block may be overwritten after this returns (+ __syncwarp).
__device__ __forceinline__ void store_bf16_block(const uint8_t* buf, __nv_bfloat16* dst, uint64_t ld,
                                                 uint32_t lane) {
  const uint32_t c = lane & 3;
#pragma unroll
  for (uint32_t i = 0; i < 4; ++i) {
    const uint32_t r = 8 * i + (lane >> 2);
    const uint4 v = *reinterpret_cast<const uint4*>(buf + r * 64 + ((c ^ ((r >> 1) & 3)) * 16));
    *reinterpret_cast<uint4*>(dst + (uint64_t)r * ld + c * 8) = v;
  }
  __syncwarp();
}

// order-preserving float -> uint32 key (larger score, larger key)
__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float funkey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// Largest key `lo` with #{entries with key >= lo} > limit (warp-cooperative, all lanes return
// it); entries (score, id) are read through get(e), e < total.
template <typename Get>
__device__ __forceinline__ uint32_t warp_cut_key(Get get, uint32_t total, uint32_t limit,
                                                 uint32_t lane) {
  uint32_t lo = 0, hi = 0xffffffffu;
#pragma unroll 1
  while (lo < hi) {
    const uint32_t mid = (uint32_t)(((uint64_t)lo + hi + 1) >> 1);
    uint32_t c = 0;
    for (uint32_t e = lane; e < total; e += 32) c += fkey(get(e).x) >= mid;
    c = warp_sum(c);
    if (c > limit) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// A cut T over the n entries rp[] (all scoring above lo) with kp/2 <= #(> T) <= kp when the
// scores allow (bisection in score space; at most kp entries above T in every case), so that
// compactions free at least half the region while keeping the best kp/2.  Warp-cooperative;
// regions of up to 32 * kCutRegs entries are bisected in registers (one pass over memory).
constexpr int kCutRegs = 16;
__device__ __noinline__ float warp_cut_band(const float2* __restrict__ rp, uint32_t n, float lo,
                                            uint32_t kp, uint32_t lane) {
  if (n <= 32u * kCutRegs) {
    float r[kCutRegs];
    float hi = -INFINITY, mn = INFINITY;
#pragma unroll
    for (int i = 0; i < kCutRegs; ++i) {
      const uint32_t e = lane + 32u * i;
      r[i] = e < n ? rp[e].x : -INFINITY;
      hi = fmaxf(hi, r[i]);
      if (e < n) mn = fminf(mn, r[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      hi = fmaxf(hi, __shfl_xor_sync(XKNN_FULL_MASK, hi, o));
      mn = fminf(mn, __shfl_xor_sync(XKNN_FULL_MASK, mn, o));
    }
    // invariant: #(> lo) > kp, #(> hi) <= kp; the first compaction of a unit starts from the
    // region's minimum
    if (!(lo > -INFINITY)) lo = nextafterf(mn, -INFINITY);
#pragma unroll 1
    for (int it = 0; it < 40; ++it) {
      const float mid = 0.5f * (lo + hi);
      if (!(mid > lo && mid < hi)) break;  // adjacent floats
      uint32_t c = 0;
#pragma unroll
      for (int i = 0; i < kCutRegs; ++i) c += r[i] > mid;
      c = warp_sum(c);
      if (c > kp) {
        lo = mid;
      } else {
        hi = mid;
        if (2 * c >= kp) break;
      }
    }
    return hi;
  }
  float hi = -INFINITY;
  for (uint32_t e = lane; e < n; e += 32) hi = fmaxf(hi, rp[e].x);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hi = fmaxf(hi, __shfl_xor_sync(XKNN_FULL_MASK, hi, o));
  if (!(lo > -INFINITY)) {
    float mn = INFINITY;
    for (uint32_t e = lane; e < n; e += 32) mn = fminf(mn, rp[e].x);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(XKNN_FULL_MASK, mn, o));
    lo = nextafterf(mn, -INFINITY);
  }
#pragma unroll 1
  for (int it = 0; it < 40; ++it) {
    const float mid = 0.5f * (lo + hi);
    if (!(mid > lo && mid < hi)) break;
    uint32_t c = 0;
    for (uint32_t e = lane; e < n; e += 32) c += rp[e].x > mid;
    c = warp_sum(c);
    if (c > kp) {
      lo = mid;
    } else {
      hi = mid;
      if (2 * c >= kp) break;
    }
  }
  return hi;
}

constexpr int kMergeRegs = 36;  // merges of up to 32 * 36 entries bisect in registers

// Merge of one row's persistent candidate list with the two regions of its unit slot: the cut
// becomes the largest of the three cuts (every column left out of any of them scores <= it).
// Common case (late column chunks): neither region raised its cut and the new entries fit the
// list's spare capacity -- they are appended.  Otherwise the entries above the cut are kept,
// and if more than kcap remain the cut rises to the (kprime+1)-th largest score (at most kprime
// kept), leaving kcap - kprime slots for the next appends.
// Invariant: every column not in the list has approx score <= lcut[row].
__device__ __noinline__ void merge_candidates(float2* __restrict__ list, uint32_t* __restrict__ lcnt,
                                              float* __restrict__ lcut,
                                              const float2* __restrict__ cand,
                                              const uint32_t* __restrict__ cnt,
                                              const float* __restrict__ tau, uint32_t ch,
                                              uint32_t kp, uint32_t kcap, uint32_t row,
                                              uint32_t slot, uint32_t lane) {
  const uint32_t n0 = cnt[slot * 2], n1 = cnt[slot * 2 + 1];
  if (n0 + n1 == 0) return;  // nothing new: the regions' cuts never rose above lcut
  float2* L = list + (uint64_t)row * kcap;
  const float2* R0 = cand + (uint64_t)slot * 2 * ch;
  const float2* R1 = R0 + ch;
  const uint32_t nl = lcnt[row];
  const float lc = lcut[row];
  float T = fmaxf(lc, fmaxf(tau[slot * 2], tau[slot * 2 + 1]));
  const uint32_t total = nl + n0 + n1;
  if (T == lc && total <= kcap) {  // every region entry scores > lc: append
    for (uint32_t e = lane; e < n0 + n1; e += 32) L[nl + e] = e < n0 ? R0[e] : R1[e - n0];
    if (lane == 0) lcnt[row] = total;
    return;
  }
  auto get = [&](uint32_t e) -> float2 {
    return e < nl ? L[e] : (e < nl + n0 ? R0[e - nl] : R1[e - nl - n0]);
  };
  if (total <= 32u * kMergeRegs) {  // keys in registers: one pass over memory, then bisection
    uint32_t key[kMergeRegs];
    const uint32_t tk = fkey(T);
    uint32_t above = 0;
#pragma unroll
    for (int i = 0; i < kMergeRegs; ++i) {
      const uint32_t e = lane + 32u * i;
      key[i] = e < total ? fkey(get(e).x) : 0u;  // 0: below every score's key
      above += key[i] > tk;
    }
    above = warp_sum(above);
    if (above > kcap) {  // largest key lo with #(>= lo) > kp; keep the entries above it
      uint32_t lo = tk, hi = 0xffffffffu;
#pragma unroll 1
      while (lo < hi) {
        const uint32_t mid = (uint32_t)(((uint64_t)lo + hi + 1) >> 1);
        uint32_t c = 0;
#pragma unroll
        for (int i = 0; i < kMergeRegs; ++i) c += key[i] >= mid;
        c = warp_sum(c);
        if (c > kp) lo = mid; else hi = mid - 1;
      }
      T = funkey(lo);
    }
  } else {
    uint32_t above = 0;
    for (uint32_t e = lane; e < total; e += 32) above += get(e).x > T;
    above = warp_sum(above);
    if (above > kcap) T = funkey(warp_cut_key(get, total, kp, lane));
  }
  uint32_t w = 0;
  for (uint32_t base = 0; base < total; base += 32) {
    const uint32_t e = base + lane;
    const float2 v = e < total ? get(e) : make_float2(-INFINITY, 0.f);
    const bool keep = e < total && v.x > T;
    __syncwarp();  // this chunk is read before any of it is overwritten (w <= base)
    const uint32_t bal = __ballot_sync(XKNN_FULL_MASK, keep);
    if (keep) L[w + __popc(bal & ((1u << lane) - 1))] = v;
    w += __popc(bal);
    __syncwarp();
  }
  if (lane == 0) {
    lcnt[row] = w;
    lcut[row] = T;
  }
}

// Region full: the new cut is the kprime-th largest score; keep the entries strictly above it.
// Every dropped (and every later rejected) column has approx score <= the returned cut.
template <int KIND, int MCP = 1>
__global__ void __launch_bounds__(384, 1)
    k_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const __grid_constant__ CUtensorMap tmOut, const __grid_constant__ CUtensorMap tmOut2,
            GemmArgs a) {
  using C = Cfg2<KIND>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned by pointer arithmetic on the __shared__ array, so the compiler keeps the
  // shared address space (STS/LDS for the epilogue staging, not generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (uint32_t)(reinterpret_cast<uintptr_t>(smem_raw) & 1023u)) & 1023u);
  uint8_t* sRes = smem;                                      // F: resident A
  uint8_t* sA = sRes + C::ARES_BYTES;                        // staged A
  uint8_t* sB = sA + C::STAGES * C::A_BYTES;                 // staged B
  uint8_t* sStg = sB + C::STAGES * C::B_BYTES;               // epilogue staging, 8 warps
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStg + 8 * C::NSTG * C::STG);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* afull = tempty + 2;
  uint64_t* aempty = afull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 1);
  // kG: each column half's current cut per row, [half][row]; the other half may use it too
  float* shcut = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);
  if (KIND == kG) shcut[threadIdx.x & 255] = -INFINITY;  // 384 threads cover the 256 slots

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // cluster of 2 * MCP CTAs: MCP CTA pairs; cta = rank in the pair, pc = pair in the cluster
  const uint32_t crank = tc::cluster_ctarank();
  const uint32_t cta = crank & 1, pc = crank >> 1, lead = crank & ~1u;
  const bool leader = cta == 0;
  const uint16_t pmask = (uint16_t)(3u << (2 * pc));        // this pair's CTAs
  const uint16_t cmask = (uint16_t)((1u << (2 * MCP)) - 1);  // every CTA of the cluster
  const uint16_t bmask = (uint16_t)((1u << cta) | (1u << (cta + 2)));  // B multicast (MCP = 2)
  // unit stream: one per cluster (its pairs take sibling units)
  const uint32_t pair = blockIdx.x / (2 * MCP), npairs = gridDim.x / (2 * MCP);

  if (warp == 0 && lane == 0) {
    for (uint32_t s = 0; s < C::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], MCP);  // a stage is free once every pair's MMAs consumed it
    }
    for (uint32_t s = 0; s < 2; ++s) {
      tc::mbar_init(&tfull[s], 1);
      tc::mbar_init(&tempty[s], 16);  // 8 epilogue warps in each CTA of the pair
    }
    tc::mbar_init(afull, 1);
    tc::mbar_init(aempty, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    tc::tma_prefetch(&tmOut);
  }
  if (warp == 2) tc::tmem_alloc_2sm<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();  // peers see initialised barriers before any remote arrive / TMA
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;
  griddep_wait();  // the setup above overlapped the previous kernel's tail (PDL)

  const uint32_t mw = KIND == kG ? a.nrows : a.st->active_count;
  const uint32_t nunits = num_units2<KIND, MCP>(a, mw);

  if (warp == 0) {
    // ================= TMA producer (both CTAs load their half) =================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, aphase = 0;
      for (uint32_t u = pair; u < nunits; u += npairs) {
        const Unit2 x = unit2_of<KIND, MCP>(a, mw, u, pc);
        if (!x.valid) continue;
        const int32_t myrow = (int32_t)(x.row0 + cta * 128);
        uint32_t nk;
        if (KIND == kF || KIND == kG) {
          tc::mbar_wait(aempty, aphase ^ 1);
          aphase ^= 1;
          if (leader) tc::mbar_expect_tx(afull, 2 * C::ARES_BYTES);
#pragma unroll 1
          for (int kc = 0; kc < 8; ++kc)
            tc::tma_load_2d_2sm(sRes + kc * 16384, &tmA, afull, kc * 64, myrow);
          nk = (x.t1 - x.t0) * 8;
        } else {
          nk = x.t1 - x.t0;
        }
        for (uint32_t k = 0; k < nk; ++k) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          if (leader) tc::mbar_expect_tx(&full[stage], 2 * (C::A_BYTES + C::B_BYTES));
          uint8_t* dA = sA + stage * C::A_BYTES;
          uint8_t* dB = sB + stage * C::B_BYTES;
          if (KIND == kF || KIND == kG) {
            const uint32_t ct = x.t0 + k / 8, kc = k % 8;
            if (MCP == 1)
              tc::tma_load_2d_2sm(dB, &tmB, &full[stage], (int32_t)(kc * 64),
                                  (int32_t)(ct * 256 + cta * 128));
            else  // this pair fetches 64 of the 128 rows for both pairs (tmB box: 64 rows)
              tc::tma_load_2d_2sm_mc(dB + pc * 8192, &tmB, &full[stage], (int32_t)(kc * 64),
                                     (int32_t)(ct * 256 + cta * 128 + pc * 64), bmask);
          } else {
            constexpr uint32_t KC = KIND == kDX ? Cfg2<kDX>::KC : Cfg2<kDW>::KC;
            constexpr uint32_t BOX = 64 * KC * 2;  // one MN-major atom (64 columns x KC rows)
            const int32_t kk = (int32_t)((x.t0 + k) * KC);
            if (KIND == kDX) {
              tc::tma_load_2d_2sm(dA, &tmA, &full[stage], kk, myrow);  // P~ [b][class]
            } else {
#pragma unroll
              for (int j = 0; j < 2; ++j)  // P~ᵀ: this CTA's 128 classes at batch rows kk..
                tc::tma_load_2d_2sm(dA + j * BOX, &tmA, &full[stage], myrow + j * 64, kk);
            }
            if (MCP == 1 || KIND == kDW) {
#pragma unroll
              for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h)  // this CTA's half of each 256-wide N instruction
                  tc::tma_load_2d_2sm(dB + (j * 2 + h) * BOX, &tmB, &full[stage],
                                      (int32_t)(256 * j + 128 * cta + 64 * h), kk);
            } else {  // pair pc fetches the h = pc pieces for both pairs
#pragma unroll
              for (int j = 0; j < 2; ++j)
                tc::tma_load_2d_2sm_mc(dB + (j * 2 + pc) * BOX, &tmB, &full[stage],
                                       (int32_t)(256 * j + 128 * cta + 64 * pc), kk, bmask);
            }
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA, one thread) =================
    if (leader && lane == 0) {
      uint32_t stage = 0, phase = 0, buf = 0, tphase = 0, aphase = 0;
      for (uint32_t u = pair; u < nunits; u += npairs) {
        const Unit2 x = unit2_of<KIND, MCP>(a, mw, u, pc);
        if (!x.valid) continue;
        const uint32_t ntile = (KIND == kF || KIND == kG) ? x.t1 - x.t0 : 1;
        if (KIND == kF || KIND == kG) {
          tc::mbar_wait(afull, aphase);
          aphase ^= 1;
        }
        for (uint32_t t = 0; t < ntile; ++t) {
          tc::mbar_wait(&tempty[buf], tphase ^ 1);
          tc::fence_after_sync();
          const uint32_t dcol = tbase + buf * C::ACC;
          const uint32_t nk = (KIND == kF || KIND == kG) ? 8 : x.t1 - x.t0;
          for (uint32_t k = 0; k < nk; ++k) {
            tc::mbar_wait(&full[stage], phase);
            tc::fence_after_sync();
            const uint32_t a0 = tc::smem_u32(sA + stage * C::A_BYTES);
            const uint32_t b0 = tc::smem_u32(sB + stage * C::B_BYTES);
            if (KIND == kF || KIND == kG) {
              constexpr uint32_t id = KIND == kG ? tc::idesc_f16(256, 256, false, false)
                                                 : tc::idesc_bf16(256, 256, false, false);
              const uint32_t r0 = tc::smem_u32(sRes + k * 16384);
#pragma unroll
              for (uint32_t kk = 0; kk < 4; ++kk)
                tc::mma_bf16_2sm(dcol, tc::smem_desc(r0 + kk * 32, 16, 1024, tc::kSwizzle128),
                                 tc::smem_desc(b0 + kk * 32, 16, 1024, tc::kSwizzle128), id,
                                 (k | kk) != 0);
            } else {
              constexpr uint32_t id = tc::idesc_bf16(256, 256, KIND == kDW, true);
              constexpr uint32_t KC = KIND == kDX ? Cfg2<kDX>::KC : Cfg2<kDW>::KC;
              constexpr uint32_t BOX = 64 * KC * 2;
#pragma unroll
              for (uint32_t kk = 0; kk < KC / 16; ++kk) {
                const uint64_t da =
                    KIND == kDX
                        ? (KC == 64 ? tc::smem_desc(a0 + kk * 32, 16, 1024, tc::kSwizzle128)
                                    : tc::smem_desc(a0 + kk * 32, 16, 512, tc::kSwizzle64))
                        : tc::smem_desc(a0 + kk * 2048, BOX, 1024, tc::kSwizzle128);
#pragma unroll
                for (uint32_t j = 0; j < 2; ++j)
                  tc::mma_bf16_2sm(dcol + j * 256, da,
                                   tc::smem_desc(b0 + j * 2 * BOX + kk * 2048, BOX, 1024,
                                                 tc::kSwizzle128),
                                   id, (k | kk) != 0);
              }
            }
            tc::mma_commit_2sm(&empty[stage], cmask);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
          if (nk) tc::mma_commit_2sm(&tfull[buf], pmask);
          else { tc::mbar_arrive_remote(&tfull[buf], lead); tc::mbar_arrive_remote(&tfull[buf], lead + 1); }
          if (++buf == C::NBUF) { buf = 0; tphase ^= 1; }
        }
        if (KIND == kF || KIND == kG) tc::mma_commit_2sm(aempty, pmask);  // A may be replaced
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue (both CTAs: their own 128 rows) =================
    const uint32_t q = warp & 3, h = (warp - 4) >> 2, ew = warp - 4;
    const uint32_t row = q * 32 + lane;
    const uint32_t lane_addr = (q * 32) << 16;
    uint8_t* stg = sStg + ew * C::NSTG * C::STG;
    uint32_t sbuf = 0;
    uint32_t buf = 0, tphase = 0;
    auto stage_flush = [&](int32_t c0, int32_t r0) {
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tc::tma_store_2d(&tmOut, stg + sbuf * C::STG, c0, r0);
        tc::tma_store_commit();
      }
      sbuf = sbuf + 1 == C::NSTG ? 0 : sbuf + 1;
      if (lane == 0) tc::tma_store_wait_read<(C::NSTG > 1 ? (int)C::NSTG - 1 : 0)>();  // next buffer free
      __syncwarp();
    };
    for (uint32_t u = pair; u < nunits; u += npairs) {
      const Unit2 x = unit2_of<KIND, MCP>(a, mw, u, pc);
      if (!x.valid) continue;
      const uint32_t ntile = (KIND == kF || KIND == kG) ? x.t1 - x.t0 : 1;
      // kG: this thread's (row, column half) candidate region state for the whole unit
      const uint32_t grow = x.row0 + cta * 128 + row;
      const uint32_t slot = (blockIdx.x >> 1) * 256 + cta * 128 + row;
      float2* creg = KIND == kG ? a.cand + ((uint64_t)slot * 2 + h) * a.ch : nullptr;
      uint32_t ccnt = 0;
      float ctau = -INFINITY;
      if (KIND == kG && grow < a.nrows) ctau = a.lcut[grow];
      for (uint32_t t = 0; t < ntile; ++t) {
        tc::mbar_wait(&tfull[buf], tphase);
        tc::fence_after_sync();
        const uint32_t tb = tbase + buf * C::ACC + lane_addr;
        const int32_t grow0 = (int32_t)(x.row0 + cta * 128 + q * 32);  // this warp's 32 rows
        if (KIND == kG) {
          // threshold top-k' of approximate scores: insert columns above the current cut;
          // when the region fills, raise the cut to its kprime-th largest score and compact
          const bool vrow = grow < a.nrows;
          const uint32_t cap = a.ch, kp = a.kprime;
          auto gproc = [&](const uint32_t (&r)[32], uint32_t chk) {
            const uint32_t col = h * 128 + chk * 32;
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            const uint32_t c0 = (x.t0 + t) * 256 + col;
            // the common case late in the scan: nothing in the warp's 32x32 chunk beats its
            // cut -- one max tree and a vote instead of 32 compares per lane
            // the other half's cut is a valid cut for this half too (the merge takes the max)
            ctau = fmaxf(ctau, shcut[(h ^ 1) * 128 + row]);
            float mx = v[0];
#pragma unroll
            for (int j = 1; j < 31; j += 2) mx = fmaxf(mx, fmaxf(v[j], v[j + 1]));
            mx = fmaxf(mx, v[31]);
            if (!__any_sync(XKNN_FULL_MASK, vrow && mx > ctau)) return;
            uint32_t mask = 0;  // columns of this chunk above the current cut
#pragma unroll
            for (int j = 0; j < 32; ++j) mask |= (v[j] > ctau ? 1u : 0u) << j;
            // columns past the block's end and the row itself never enter
            if (!vrow) mask = 0;
            if (c0 + 32 > a.ncols) mask &= a.ncols > c0 ? (0xffffffffu >> (32 - (a.ncols - c0))) : 0u;
            const uint32_t selfc = a.row_base + grow - a.col_base - c0;  // self column in chunk
            if (selfc < 32) mask &= ~(1u << selfc);
            if (!__any_sync(XKNN_FULL_MASK, mask != 0)) return;
            if (__reduce_max_sync(XKNN_FULL_MASK, (uint32_t)__popc(mask)) >= 8 &&
                __all_sync(XKNN_FULL_MASK, ccnt + __popc(mask) <= cap)) {
              // dense chunk (early in a scan), every lane's columns fit its region: one
              // predicated store per column instead of a divergent per-lane loop whose trip
              // count is the warp's largest popcount
              float2* dst = creg + ccnt;
              uint32_t wi = 0;
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if ((mask >> j) & 1u) dst[wi++] = make_float2(v[j], __uint_as_float(a.col_base + c0 + j));
              ccnt += wi;
              return;
            }
            float sc[32];  // spill-friendly copy for the dynamic-index inserts
#pragma unroll
            for (int j = 0; j < 32; ++j) sc[j] = v[j];
            // warp-synchronous insertion: each round every lane inserts its next column above
            // the cut; lanes whose region is full are compacted by the whole warp in turn
            // (a lane-serial compaction would diverge the warp 32 ways)
#pragma unroll 1
            while (__any_sync(XKNN_FULL_MASK, mask != 0)) {
              bool full = false;
              if (mask) {
                const int j = __ffs(mask) - 1;
                const float sj = sc[j];
                if (!(sj > ctau)) {
                  mask &= mask - 1;
                } else if (ccnt < cap) {
                  creg[ccnt++] = make_float2(sj, __uint_as_float(a.col_base + c0 + j));
                  mask &= mask - 1;
                } else {
                  full = true;  // bit j stays set: retried after the compaction
                }
              }
              uint32_t fb = __ballot_sync(XKNN_FULL_MASK, full);
              while (fb) {
                const int f = __ffs(fb) - 1;
                fb &= fb - 1;
                float2* rp = reinterpret_cast<float2*>(
                    __shfl_sync(XKNN_FULL_MASK, reinterpret_cast<unsigned long long>(creg), f));
                const uint32_t n = __shfl_sync(XKNN_FULL_MASK, ccnt, f);
                // new cut: a score with between kp/2 and kp entries above it (bisection in
                // score space from [old cut, max]); the entries above it are kept
                const float T = warp_cut_band(rp, n, __shfl_sync(XKNN_FULL_MASK, ctau, f), kp,
                                              lane);
                uint32_t w = 0;
                for (uint32_t base = 0; base < n; base += 32) {
                  const uint32_t e = base + lane;
                  const float2 x = e < n ? rp[e] : make_float2(-INFINITY, 0.f);
                  const bool keep = e < n && x.x > T;
                  __syncwarp();
                  const uint32_t bal = __ballot_sync(XKNN_FULL_MASK, keep);
                  if (keep) rp[w + __popc(bal & ((1u << lane) - 1))] = x;
                  w += __popc(bal);
                  __syncwarp();
                }
                if ((int)lane == f) {
                  ctau = T;
                  ccnt = w;
                  shcut[h * 128 + row] = T;
                }
              }
            }
          };
          // the next chunk's TMEM load is in flight while this one is scanned; TMEM is released
          // as soon as the last chunk is in registers
          uint32_t ra[32], rb[32];
          tc::tmem_ld32_issue(tb + h * 128, ra);
          tc::tmem_ld_wait(ra);
          tc::tmem_ld32_issue(tb + h * 128 + 32, rb);
          gproc(ra, 0);
          tc::tmem_ld_wait(rb);
          tc::tmem_ld32_issue(tb + h * 128 + 64, ra);
          gproc(rb, 1);
          tc::tmem_ld_wait(ra);
          tc::tmem_ld32_issue(tb + h * 128 + 96, rb);
          gproc(ra, 2);
          tc::tmem_ld_wait(rb);
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_remote_relaxed(&tempty[buf], lead);
          gproc(rb, 3);
          if (t + 1 == ntile) {
            a.cnt[slot * 2 + h] = ccnt;
            a.tau[slot * 2 + h] = ctau;
          }
        } else if (KIND == kF) {
          const uint32_t ct = x.t0 + t;
          const uint32_t b = x.row0 + cta * 128 + row;
          const bool vrow = b < a.B;
          const int32_t lc = vrow ? a.label_col[b] : -1;
          const float k2 = a.scale * 1.4426950408889634f;
          float sum = 0.f, lab = 0.f;
          bool has = false;
          auto process = [&](const uint32_t (&r)[32], uint32_t ch) {
            const uint32_t col = h * 128 + ch * 32;
            const uint32_t c0 = ct * 256 + col;
            uint32_t pk[16];
            if (vrow && c0 + 32 <= mw) {  // interior chunk: 1 FFMA + 1 MUFU.EX2 + 1 FADD each
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float e0 = ex2_approx(fmaf(__uint_as_float(r[j]), k2, -k2));
                const float e1 = ex2_approx(fmaf(__uint_as_float(r[j + 1]), k2, -k2));
                sum += e0;
                sum += e1;
                pk[j / 2] = pack_bf16(e0, e1);
              }
            } else {  // ragged edge: padded classes / batch rows contribute exact zeros
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const bool ok0 = vrow && c0 + j < mw, ok1 = vrow && c0 + j + 1 < mw;
                const float e0 = ok0 ? ex2_approx(fmaf(__uint_as_float(r[j]), k2, -k2)) : 0.f;
                const float e1 =
                    ok1 ? ex2_approx(fmaf(__uint_as_float(r[j + 1]), k2, -k2)) : 0.f;
                sum += e0;
                sum += e1;
                pk[j / 2] = pack_bf16(e0, e1);
              }
            }
            if (lc >= (int32_t)c0 && lc < (int32_t)c0 + 32) {  // at most once per row
              const int32_t idx = lc - (int32_t)c0;
              float sel = 0.f;
#pragma unroll
              for (int j = 0; j < 32; ++j) sel = (j == idx) ? __uint_as_float(r[j]) : sel;
              lab = sel * a.scale;
              has = true;
            }
            stage_bf16(stg, lane, pk);
            __syncwarp();
            store_bf16_block(stg, a.Pt + (uint64_t)grow0 * a.ldp + c0, a.ldp, lane);
          };
          // the next chunk's TMEM load is in flight while this one is exponentiated and
          // stored; TMEM is released as soon as the last chunk is in registers
          uint32_t ra[32], rb[32];
          tc::tmem_ld32_issue(tb + h * 128, ra);
          tc::tmem_ld_wait(ra);
          tc::tmem_ld32_issue(tb + h * 128 + 32, rb);
          process(ra, 0);
          tc::tmem_ld_wait(rb);
          tc::tmem_ld32_issue(tb + h * 128 + 64, ra);
          process(rb, 1);
          tc::tmem_ld_wait(ra);
          tc::tmem_ld32_issue(tb + h * 128 + 96, rb);
          process(ra, 2);
          tc::tmem_ld_wait(rb);
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_remote_relaxed(&tempty[buf], lead);
          process(rb, 3);
          a.partial[(uint64_t)(ct * 2 + h) * a.bpad + b] = sum;
          if (has) a.labelterm[b] = lab - a.scale;
        } else {
          // dX: split-K partial rows of unit x.id; dW: dW rows (compact active order), or the
          // fp32 K-partial rows of a split tail unit (slot x.id)
          const bool part = KIND == kDW && x.part;
          const int32_t orow = (KIND == kDX || part) ? (int32_t)(x.id * 256) + grow0 - (int32_t)x.row0
                                                     : grow0;
          const bool zero = KIND == kDX && x.t1 == x.t0;
#pragma unroll 1
          for (uint32_t ch = 0; ch < 8; ++ch) {
            const uint32_t col = h * 256 + ch * 32;
            float v[32];
            if (!zero) {
              tc::tmem_ld32(tb + col, v);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = 0.f;
            }
            if (KIND == kDW && part) {  // fp32 partial through the warp's whole 4 KB staging
              if (lane == 0) tc::tma_store_wait_read<0>();
              __syncwarp();
              stage_f32(stg, lane, v);
              tc::fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tc::tma_store_2d(&tmOut2, stg, (int32_t)col, orow);
                tc::tma_store_commit();
                tc::tma_store_wait_read<0>();
              }
              __syncwarp();
              continue;
            }
            if (KIND == kDW) {  // dW rows in bf16 (64-B swizzled staging rows)
              uint32_t pk[16];
#pragma unroll
              for (int j = 0; j < 32; j += 2) pk[j / 2] = pack_bf16(v[j], v[j + 1]);
              stage_bf16(stg + sbuf * C::STG, lane, pk);
            } else {
              stage_f32(stg + sbuf * C::STG, lane, v);
            }
            stage_flush((int32_t)col, orow);
          }
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_remote_relaxed(&tempty[buf], lead);
        }
        if (++buf == C::NBUF) { buf = 0; tphase ^= 1; }
      }
      if (KIND == kG) {
        // unit end: fold both column halves' regions into the rows' persistent lists; warp
        // (q, h) merges rows q*32 + 2i + h of this CTA
        epilogue_bar();
#pragma unroll 1
        for (uint32_t i = 0; i < 16; ++i) {
          const uint32_t r = q * 32 + 2 * i + h;
          const uint32_t gr = x.row0 + cta * 128 + r;
          if (gr < a.nrows)
            merge_candidates(a.list, a.lcnt, a.lcut, a.cand, a.cnt, a.tau, a.ch, a.kprime, a.kcap, gr,
                             (blockIdx.x >> 1) * 256 + cta * 128 + r, lane);
        }
        shcut[h * 128 + row] = -INFINITY;  // the next unit's rows start from their lists' cuts
        epilogue_bar();  // regions free for the next unit
      }
    }
    if (lane == 0) tc::tma_store_wait_all();
    __syncwarp();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();  // both CTAs done: no MMA reads peer smem, no remote arrive in flight
  if (warp == 2) {
    tc::fence_after_sync();
    tc::tmem_dealloc_2sm<512>(tbase);
  }
}

// ---- small fused kernels of the fast path ---------------------------------------------------

// per-row softmax statistics from the GEMM-F tile partials: 32 rows x 32 tile groups per block,
// each thread sums its tile group in order, then a fixed-order combine (deterministic)
__global__ void k_rowreduce(const SelState* st, const float* __restrict__ partial,
                            const float* __restrict__ labelterm, const int32_t* __restrict__ lcol,
                            uint32_t B, uint32_t bpad, double* __restrict__ red) {
  // 8 rows x 128 tile groups per 1024-thread block (B/8 blocks: enough of them to spread the
  // partial-sum reads over the SMs); fixed summation order (deterministic)
  griddep_wait();
  griddep_launch();
  __shared__ double part[128][9];
  const uint32_t nt = 2 * ((st->active_count + 255) / 256);
  const uint32_t tx = threadIdx.x & 7, ty = threadIdx.x >> 3;  // row in block, tile group
  const uint32_t b = blockIdx.x * 8 + tx;
  double s = 0.0;
  if (b < B) {
    double s2[2] = {0.0, 0.0};
    uint32_t t = ty;
    for (; t + 128 < nt; t += 256) {
      s2[0] += (double)partial[(uint64_t)t * bpad + b];
      s2[1] += (double)partial[(uint64_t)(t + 128) * bpad + b];
    }
    for (; t < nt; t += 128) s2[0] += (double)partial[(uint64_t)t * bpad + b];
    s = s2[0] + s2[1];
  }
  part[ty][tx] = s;
  __syncthreads();
  double g = 0.0;  // threads ty < 8: row tx, groups ty*16 .. ty*16+15
  if (ty < 8)
    for (int i = 0; i < 16; ++i) g += part[ty * 16 + i][tx];
  __syncthreads();
  if (ty < 8) part[ty][tx] = g;
  __syncthreads();
  if (ty == 0 && b < B) {
    double tot = 0.0;
    for (int g2 = 0; g2 < 8; ++g2) tot += part[g2][tx];
    const int32_t c = lcol[b];
    red[b] = tot;
    red[B + b] = c >= 0 ? (double)labelterm[b] : 0.0;
    red[2 * B + b] = c >= 0 ? 1.0 : 0.0;
  }
}

// X_hat' = bf16(x_hat * s / (B * sum)); pad rows zeroed; the batch rows of every local label
// column linked into lists (lab_head[col] -> lab_next[b] -> ..., -1 terminated; the row update
// consumes and clears them)
template <int DV>
__global__ void k_fixup(const double* __restrict__ red, const int32_t* __restrict__ lcol,
                        const float* __restrict__ X, const float* __restrict__ xnorm, uint32_t B,
                        uint32_t bpad, uint32_t d, float scale, int32_t* __restrict__ lab_head,
                        int32_t* __restrict__ lab_next, __nv_bfloat16* __restrict__ Xs,
                        double* __restrict__ loss, SelState* st, unsigned long long* err) {
  griddep_wait();
  griddep_launch();
  if (blockIdx.x == 0) {
    // the step's loss (k_loss's arithmetic, 256 threads): red is final once this grid runs
    __shared__ double part[256];
    double s = 0.0;
    const uint32_t chunk = (B + blockDim.x - 1) / blockDim.x;
    for (uint32_t i = threadIdx.x * chunk; i < min(B, (threadIdx.x + 1) * chunk); ++i) {
      if (red[2 * B + i] != 1.0) raise_error(err, XKNN_ERR_LABEL_OUT_OF_RANGE, i);
      s += log(red[i]) - red[B + i];
    }
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (uint32_t k = 0; k < blockDim.x; ++k) t += part[k];
      const double l = t / (double)B;
      *loss = l;
      st->loss = l;
    }
  }
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < bpad;
       b += (gridDim.x * blockDim.x) >> 5) {
    uint2* dst = reinterpret_cast<uint2*>(Xs + (uint64_t)b * d);
    if (b >= B) {
#pragma unroll
      for (int c = 0; c < DV; ++c) dst[lane + 32 * c] = make_uint2(0, 0);
      continue;
    }
    const double denom = red[b];
    const int32_t lc = lcol[b];
    if (lane == 0 && lc >= 0) lab_next[b] = atomicExch(&lab_head[lc], (int32_t)b);
    const float inv = 1.0f / xnorm[b];
    const float rs = (float)((double)scale / ((double)B * denom));
    const float4* xp = reinterpret_cast<const float4*>(X + (uint64_t)b * d);
#pragma unroll
    for (int c = 0; c < DV; ++c) {
      const float4 x = xp[lane + 32 * c];
      dst[lane + 32 * c] = make_uint2(pack_bf16(__fmul_rn(x.x, inv) * rs, __fmul_rn(x.y, inv) * rs),
                                      pack_bf16(__fmul_rn(x.z, inv) * rs, __fmul_rn(x.w, inv) * rs));
    }
  }
}

// dX[b][:] = s * r_b * sum_s partial[s][b][:] (fixed split order) - (s/B) * w_hat[y_b] when the
// label's class is in this shard (w_hat recomputed in fp32 from W and its cached norm, exactly as
// the gather normalized it)
__global__ void k_dx_reduce(const float* __restrict__ partial, const double* __restrict__ red,
                            uint32_t B, uint32_t nbt, uint32_t splits, uint32_t rows_per_unit,
                            float scale, const int32_t* __restrict__ lcol,
                            const uint32_t* __restrict__ active, uint64_t begin,
                            const float* __restrict__ W, const float* __restrict__ wnorm,
                            float* __restrict__ out) {
  griddep_wait();
  griddep_launch();
  const uint64_t total = (uint64_t)B * 128;  // float4 units (D = 512)
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = (uint32_t)(e / 128), c4 = (uint32_t)(e % 128);
    const uint32_t bt = b / rows_per_unit, row = b % rows_per_unit;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8  // 8 partial loads in flight per thread; the sum stays in split order
    for (uint32_t s = 0; s < splits; ++s) {
      const float4 v = reinterpret_cast<const float4*>(
          partial + ((uint64_t)(s * nbt + bt) * rows_per_unit + row) * 512)[c4];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    const float rs = (float)((double)scale / ((double)B * red[b]));
    float4 o = make_float4(acc.x * rs, acc.y * rs, acc.z * rs, acc.w * rs);
    const int32_t lc = lcol[b];
    if (lc >= 0) {
      const float sb = (float)((double)scale / (double)B);
      const float inv = 1.0f / wnorm[lc];
      const float4 w = reinterpret_cast<const float4*>(W + ((uint64_t)active[lc] - begin) * 512)[c4];
      o.x = __fsub_rn(o.x, __fmul_rn(sb, __fmul_rn(w.x, inv)));
      o.y = __fsub_rn(o.y, __fmul_rn(sb, __fmul_rn(w.y, inv)));
      o.z = __fsub_rn(o.z, __fmul_rn(sb, __fmul_rn(w.z, inv)));
      o.w = __fsub_rn(o.w, __fmul_rn(sb, __fmul_rn(w.w, inv)));
    }
    reinterpret_cast<float4*>(out + (uint64_t)b * 512)[c4] = o;
  }
}

__global__ void k_zero_rows_bf16(const SelState* st, __nv_bfloat16* W16, uint32_t cap_rows,
                                 uint32_t d) {
  griddep_wait();
  griddep_launch();
  // rows [count, round_up(count, 256)) of W_sub must be zero for the K loop of GEMM-dX
  const uint32_t c = st->active_count;
  const uint32_t e = min(cap_rows, (c + 255) / 256 * 256);
  const uint64_t n = (uint64_t)(e - c) * d / 8;
  uint4* p = reinterpret_cast<uint4*>(W16 + (uint64_t)c * d);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
}

// ---- host-side tensor maps ------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
              uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw, bool f32 = false) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
            const_cast<void*>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

struct FastState {
  uint32_t bpad = 0, mwpad = 0;
  uint64_t dx_units_cap = 0;
  float* partial_f = nullptr;       // [2 * mwpad/256][bpad]
  float* labelterm = nullptr;       // [bpad]
  float* partial_dx = nullptr;      // [units][256][512]
  __nv_bfloat16* dW16 = nullptr;    // [mwpad][512] weight gradient, compact active order
  float* dw_part = nullptr;         // [74 slots][256][512] GEMM-dW tail-unit K-partials
  int32_t* lab_head = nullptr;      // [mwpad] first batch row labelled with each active column
  int32_t* lab_next = nullptr;      // [bpad]  next batch row with the same label column
  CUtensorMap mF_A, mF2_B, mDX_A, mDX_B, mDW_A, mDW_B;
  CUtensorMap mPt_st, mDXP_st, mDW_st, mF2_B64, mDWP_st;
};

// splits per 256-row pair tile so that (pair tiles x splits) units fill the 74 CTA pairs in
// whole waves: the fewest splits with >= 95% wave efficiency (else the most efficient), at most
// max_units units
uint32_t gemm_pair_splits(uint32_t nbp, uint32_t max_units, uint32_t streams) {
  uint32_t best = 1;
  double best_eff = -1;
  for (uint32_t s = 1; s <= streams && (uint64_t)nbp * s <= max_units; ++s) {
    const uint32_t u = nbp * s;
    const double eff =
        (double)u / ((double)((u + streams - 1) / streams) * streams);
    if (eff >= 0.95) return s;
    if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
  }
  return best;
}

// CTAs of a persistent GEMM launched in clusters of `cluster`: whole clusters that can be
// co-resident (4-CTA clusters do not tile every GPC of the 148 SMs)
template <typename K>
static unsigned cluster_grid(K kernel, unsigned cluster, size_t smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kNumSMs);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess || n <= 0) {
    (void)cudaGetLastError();
    return kNumSMs / cluster * cluster;
  }
  return std::min<unsigned>((unsigned)n * cluster, kNumSMs / cluster * cluster);
}

cudaError_t launch_rowreduce(const SelState* st, const float* partial, const float* labelterm,
                             const int32_t* lcol, uint32_t B, uint32_t bpad, double* red,
                             cudaStream_t s) {
  launch_pdl(k_rowreduce, (unsigned)((B + 7) / 8), 1024, 0, s, st, partial, labelterm, lcol, B,
             bpad, red);
  return cudaGetLastError();
}

cudaError_t launch_dx_reduce(const float* partial, const double* red, uint32_t B, uint32_t nbt,
                             uint32_t splits, float scale, const int32_t* lcol,
                             const uint32_t* active, uint64_t begin, const float* W,
                             const float* wnorm, float* out, cudaStream_t s) {
  launch_pdl(k_dx_reduce, grid_for((uint64_t)B * 128, 256), 256, 0, s, partial, red, B, nbt,
             splits, 256u, scale, lcol, active, begin, W, wnorm, out);
  return cudaGetLastError();
}

xknn_status_t Layer::init_fast() {
  auto* f = new FastState;
  fast = f;
  if (d != 512) return fail_msg(XKNN_ERR_UNSUPPORTED, "BF16 path is specialised for D = 512");
  f->bpad = (uint32_t)((bmax + 255) / 256 * 256);
  f->mwpad = (uint32_t)((mw_cap + 255) / 256 * 256);
  ldp = f->mwpad;
  XK_CUDA(dalloc(&Xhat16, (uint64_t)f->bpad * d));
  XK_CUDA(dalloc(&Xs16, (uint64_t)f->bpad * d));
  XK_CUDA(cudaMemsetAsync(Xhat16, 0, (uint64_t)f->bpad * d * 2, stream));
  XK_CUDA(dalloc(&Wsub16, (uint64_t)f->mwpad * d));
  XK_CUDA(cudaMemsetAsync(Wsub16, 0, (uint64_t)f->mwpad * d * 2, stream));
  XK_CUDA(dalloc(&Pt, (uint64_t)f->bpad * ldp));
  XK_CUDA(cudaMemsetAsync(Pt, 0, (uint64_t)f->bpad * ldp * 2, stream));
  XK_CUDA(dalloc(&f->partial_f, (uint64_t)2 * (f->mwpad / 256) * f->bpad));
  XK_CUDA(dalloc(&f->labelterm, f->bpad));
  f->dx_units_cap = 148ull * 256;  // pair-tile units x 256 rows (at most 148 units)
  XK_CUDA(dalloc(&f->partial_dx, f->dx_units_cap * 512));
  XK_CUDA(dalloc(&f->dW16, (uint64_t)f->mwpad * d));
  XK_CUDA(dalloc(&f->dw_part, (uint64_t)kNumSMs / 2 * 256 * 512));
  XK_CUDA(dalloc(&f->lab_head, f->mwpad));
  XK_CUDA(cudaMemsetAsync(f->lab_head, 0xff, (uint64_t)f->mwpad * 4, stream));  // all -1
  XK_CUDA(dalloc(&f->lab_next, f->bpad));
  XK_CUDA(dalloc(&dXpart, (uint64_t)f->bpad * d));
  bool ok = true;
  ok &= make_map(&f->mF_A, Xhat16, d, f->bpad, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&f->mF2_B, Wsub16, d, f->mwpad, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&f->mF2_B64, Wsub16, d, f->mwpad, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B);
  constexpr uint32_t KC = Cfg2<kDX>::KC;
  ok &= make_map(&f->mDX_A, Pt, ldp, f->bpad, KC, 128,
                 KC == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
  ok &= make_map(&f->mDX_B, Wsub16, d, f->mwpad, 64, KC, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&f->mDW_A, Pt, ldp, f->bpad, 64, Cfg2<kDW>::KC, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&f->mDW_B, Xs16, d, f->bpad, 64, Cfg2<kDW>::KC, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&f->mPt_st, Pt, ldp, f->bpad, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  ok &= make_map(&f->mDXP_st, f->partial_dx, 512, f->dx_units_cap, 32, 32,
                 CU_TENSOR_MAP_SWIZZLE_128B, true);
  ok &= make_map(&f->mDW_st, f->dW16, 512, f->mwpad, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  ok &= make_map(&f->mDWP_st, f->dw_part, 512, (uint64_t)kNumSMs / 2 * 256, 32, 32,
                 CU_TENSOR_MAP_SWIZZLE_128B, true);
  if (!ok) return fail_msg(XKNN_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  XK_CUDA(cudaFuncSetAttribute(k_gemm2<kF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes2<kF>()));
  XK_CUDA(cudaFuncSetAttribute(k_gemm2<kDX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes2<kDX>()));
  XK_CUDA(cudaFuncSetAttribute(k_gemm2<kF, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes2<kF>()));
  XK_CUDA(cudaFuncSetAttribute(k_gemm2<kDX, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes2<kDX>()));
  XK_CUDA(cudaFuncSetAttribute(k_gemm2<kDW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes2<kDW>()));
  return XKNN_OK;
}

void Layer::free_fast() {
  auto* f = static_cast<FastState*>(fast);
  if (!f) return;
  if (f->partial_f) cudaFree(f->partial_f);
  if (f->labelterm) cudaFree(f->labelterm);
  if (f->partial_dx) cudaFree(f->partial_dx);
  if (f->dW16) cudaFree(f->dW16);
  if (f->lab_head) cudaFree(f->lab_head);
  if (f->lab_next) cudaFree(f->lab_next);
  if (f->dw_part) cudaFree(f->dw_part);
  delete f;
  fast = nullptr;
}

// after a failed step (device error word set): the label lists may hold entries of columns the
// aborted update never visited
xknn_status_t Layer::reset_fast_scratch() {
  auto* f = static_cast<FastState*>(fast);
  if (!f) return XKNN_OK;
  XK_CUDA(cudaMemsetAsync(f->lab_head, 0xff, (uint64_t)f->mwpad * 4, stream));
  return XKNN_OK;
}

xknn_status_t Layer::run_fast_core(uint64_t B) {
  auto* f = static_cast<FastState*>(fast);
  const uint32_t D = (uint32_t)d;
  if (B > f->bpad) return XKNN_ERR_INVALID_ARGUMENT;
  // (a) operands: gathered, normalized active rows of W (bf16) + norms -- independent of the
  //     features, so at P > 1 the feature all-gather (side stream) runs under it -- then
  //     X_hat (bf16) + norms
  XK_CUDA(launch_normalize_rows(W, mw_cap, D, active, &st->active_count, begin, nullptr, Wsub16,
                                wnorm, err, stream));
  ++launches;
  launch_pdl(k_zero_rows_bf16, 64, 256, 0, stream, st, Wsub16, f->mwpad, D);
  XK_LAUNCH();
  if (world > 1) XK_TRY(wait_features());
  XK_CUDA(launch_normalize_rows(X, B, D, nullptr, nullptr, 0, nullptr, Xhat16, xnorm, err, stream));
  ++launches;

  mark(3);
  GemmArgs ga{};
  ga.st = st;
  ga.B = (uint32_t)B;
  ga.bpad = f->bpad;
  ga.dim = D;
  ga.scale = cfg.scale;
  ga.label_col = label_col;
  ga.Pt = Pt;
  ga.ldp = ldp;
  ga.labelterm = f->labelterm;
  // (b) GEMM-F with the fused exp/row-sum/label-logit epilogue; units are (256-row pair tile,
  //     class-tile range)
  const uint32_t nbp = (uint32_t)((B + 255) / 256);
  ga.partial = f->partial_f;
  ga.nbt = nbp;
  // an even number of batch pair tiles: 4-CTA clusters, the class tiles multicast to 2 pairs
  // (opt-in, XKNN_MULTICAST=1: measured slower at C2 -- 4-CTA clusters fit on fewer SMs)
  const bool mc = (nbp % 2 == 0) && getenv("XKNN_MULTICAST");
  static const unsigned grid_f4 = cluster_grid(k_gemm2<kF, 2>, 4, smem_bytes2<kF>());
  static const unsigned grid_dx4 = cluster_grid(k_gemm2<kDX, 2>, 4, smem_bytes2<kDX>());
  if (mc) {
    ga.splits = gemm_pair_splits(nbp / 2, 1u << 30, grid_f4 / 4);
    launch_pdl_cluster(k_gemm2<kF, 2>, grid_f4, 384, smem_bytes2<kF>(), stream, 4u, f->mF_A,
                       f->mF2_B64, f->mPt_st, f->mPt_st, ga);
  } else {
    ga.splits = gemm_pair_splits(nbp, 1u << 30);
    launch_pdl_cluster(k_gemm2<kF>, kNumSMs, 384, smem_bytes2<kF>(), stream, 2u, f->mF_A,
                       f->mF2_B, f->mPt_st, f->mPt_st, ga);
  }
  XK_LAUNCH();
  mark(4);
  // (c) row statistics -> all-reduce over class shards -> loss
  launch_pdl(k_rowreduce, (unsigned)((B + 7) / 8), 1024, 0, stream, st, f->partial_f, f->labelterm, label_col,
                                                     (uint32_t)B, f->bpad, rowred);
  XK_LAUNCH();
  if (world > 1) {
    if (par_ar.ready) {  // one kernel over NVLink peer memory (peer.cu)
      XK_CUDA(par_ar.launch(rowred, 3 * B, err, stream));
      ++launches;
    } else {
      XK_NCCL(ncclAllReduce(rowred, rowred, 3 * B, ncclDouble, ncclSum, comm, stream));
    }
  }
  // (d) the row-scaled X_hat', the label lists and the loss (block 0)
  launch_pdl(k_fixup<4>, grid_for((uint64_t)f->bpad * 32, 256), 256, 0, stream, rowred, label_col,
             X, xnorm, (uint32_t)B, f->bpad, D, cfg.scale, f->lab_head, f->lab_next, Xs16,
             loss_dev, st, err);
  XK_LAUNCH();
  mark(5);
  // (e) GEMM-dW -> bf16 dW rows (compact active order)
  ga.out16 = f->dW16;
  launch_pdl_cluster(k_gemm2<kDW>, kNumSMs, 384, smem_bytes2<kDW>(), stream, 2u, f->mDW_A,
                     f->mDW_B, f->mDW_st, f->mDWP_st, ga);
  XK_LAUNCH();
  mark(6);
  // (f) GEMM-dX split-K partials -> reduce with s*r_b -> reduce-scatter over class shards
  ga.partial = f->partial_dx;
  const uint32_t dx_splits =
      mc ? gemm_pair_splits(nbp / 2, 74, grid_dx4 / 4) : gemm_pair_splits(nbp, 148);
  ga.nbt = nbp;
  ga.splits = dx_splits;
  if (mc)
    launch_pdl_cluster(k_gemm2<kDX, 2>, grid_dx4, 384, smem_bytes2<kDX>(), stream, 4u, f->mDX_A,
                       f->mDX_B, f->mDXP_st, f->mDXP_st, ga);
  else
    launch_pdl_cluster(k_gemm2<kDX>, kNumSMs, 384, smem_bytes2<kDX>(), stream, 2u, f->mDX_A,
                       f->mDX_B, f->mDXP_st, f->mDXP_st, ga);
  XK_LAUNCH();
  mark(7);
  launch_pdl(k_dx_reduce, grid_for(B * 128, 256), 256, 0, stream, f->partial_dx, rowred,
             (uint32_t)B, nbp, dx_splits, 256u, cfg.scale, (const int32_t*)label_col,
             (const uint32_t*)active, begin, (const float*)W, (const float*)wnorm,
             world > 1 ? dXpart : dX);
  XK_LAUNCH();
  const uint64_t bl = B / world;
  if (world > 1) {
    // the feature-gradient reduce-scatter over NVLink runs on the side stream, under the
    // HBM-bound row update (the only collective in flight on the communicator)
    XK_CUDA(cudaEventRecord(ev_fork, stream));
    XK_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
    XK_NCCL(ncclReduceScatter(dXpart, dX, bl * d, ncclFloat, ncclSum, comm, side));
    XK_CUDA(cudaEventRecord(ev_join, side));
  }
  // (g) normalize-backward + momentum SGD on the active rows (parallel.cpp:649-667)
  //     (a separate HBM-streaming kernel: it runs at the copy roofline, while inside the
  //     GEMM-dW kernel the few spare warps per SM could not keep enough bytes in flight)
  mark(8);
  // (the GEMM-dW tail split is off here: measured 2 us faster GEMM-dW at C2 but a 5 us slower
  // bf16 row update; on the FP32 path, whose dW is 5x longer, it pays -- fast32.cu)
  LabelFix lf{f->lab_head, f->lab_next, X, xnorm, (float)((double)cfg.scale / (double)B)};
  XK_CUDA(launch_update_rows_bf16(W, V, f->dW16, active, &st->active_count, mw_cap, begin, D,
                                  wnorm, lr_dev, cfg.momentum, cfg.weight_decay, err, stream, lf));
  ++launches;
  if (world > 1) XK_CUDA(cudaStreamWaitEvent(stream, ev_join, 0));
  return XKNN_OK;
}

}  // namespace xknn
static_assert(xknn::smem_bytes2<xknn::kF>() <= 232448, "GEMM-F pair smem");
static_assert(xknn::smem_bytes2<xknn::kDX>() <= 232448, "GEMM-dX pair smem");
static_assert(xknn::smem_bytes2<xknn::kDW>() <= 232448, "GEMM-dW pair smem");
static_assert(xknn::smem_bytes2<xknn::kG>() <= 232448, "graph GEMM pair smem");

namespace xknn {

// GEMM + threshold top-k' candidate pass of one ring hop of the graph build (graph.cu): own
// (nrows x 512 fp16, zero rows up to a multiple of 256) against the held block (ncols rows of
// global ids col_base.., buffer rows up to a multiple of 256), folded into the persistent lists.
cudaError_t launch_graph_candidates(const __half* own, uint32_t nrows, uint32_t row_base,
                                    const __half* held, uint32_t ncols, uint32_t col_base,
                                    float2* list, uint32_t* lcnt, float* lcut, uint32_t kprime,
                                    uint32_t kcap, float2* cand, uint32_t* cnt, float* tau,
                                    uint32_t ch, cudaStream_t s) {
  CUtensorMap mA, mB;
  // 4-CTA clusters: two query blocks per cluster share every class tile (multicast)
  const bool mc = nrows > 256 && getenv("XKNN_MULTICAST");
  const uint64_t apad = (nrows + 255) / 256 * 256, bpad = (ncols + 255) / 256 * 256;
  if (!make_map(&mA, own, 512, apad, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&mB, held, 512, bpad, 64, mc ? 64 : 128, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm2<kG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem_bytes2<kG>());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_gemm2<kG, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes2<kG>());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  GemmArgs ga{};
  ga.nrows = nrows;
  ga.ncols = ncols;
  ga.row_base = row_base;
  ga.col_base = col_base;
  ga.list = list;
  ga.lcnt = lcnt;
  ga.lcut = lcut;
  ga.cand = cand;
  ga.cnt = cnt;
  ga.tau = tau;
  ga.ch = ch;
  ga.kprime = kprime;
  ga.kcap = kcap;
  ga.dim = 512;
  static const uint32_t gchunk = [] {
    const char* e = getenv("XKNN_GCHUNK");  // tuning knob (class tiles per chunk)
    const long v = e ? atol(e) : 0;
    return v > 0 ? (uint32_t)v : 128u;
  }();
  ga.gchunk = gchunk;
  if (mc)
    launch_pdl_cluster(k_gemm2<kG, 2>, cluster_grid(k_gemm2<kG, 2>, 4, smem_bytes2<kG>()), 384,
                       smem_bytes2<kG>(), s, 4u, mA, mB, mA, mA, ga);
  else
    launch_pdl_cluster(k_gemm2<kG>, kNumSMs, 384, smem_bytes2<kG>(), s, 2u, mA, mB, mA, mA, ga);
  return cudaGetLastError();
}

}  // namespace xknn
