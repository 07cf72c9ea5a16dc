// fast32.cu -- XKNN_PREC_FP32: the three fc GEMMs at fp32 accuracy on 5th-gen tensor cores
// (tcgen05.mma, accumulators in TMEM, operands staged by TMA), by operand splitting.  A single
// TF32 (2^-11) or bf16 pass misses the north star's 1e-5 relative tolerance of the fp32 reference
// (matrix.cpp:57-98); each GEMM uses the cheapest split that meets it:
//   GEMM-F  (kFm, "mixed"): a_t = tf32(a);  a*b ~ a_t*b_t [kind::tf32] + bf16(a)*bf16(b - b_t)
//           + bf16(a - a_t)*bf16(b) [kind::f16] -- 2 TF32-MMA-equivalents per product; the
//           exp(s*S - s) epilogue multiplies logit errors by s = 30, so the leading product keeps
//           tf32 precision (a plain bf16x3 GEMM-F would leave 6e-6 relative errors in P~)
//   GEMM-dW (kDWh) / GEMM-dX (kDXb), "bf16x3": hi = bf16(a), lo = bf16(a - hi);  a*b ~
//           lo*hi + hi*lo + hi*hi [kind::f16] -- 1.5 TF32-equivalents; no amplification downstream
//   XKNN_FP32_GEMM=3xtf32 (kF3 / kDW3 / kDX3): hi = tf32(a), lo = a - hi;  lo*hi + hi*lo + hi*hi
//           [kind::tf32], |error| <~ 2^-21 |a*b| -- 3 TF32-equivalents ("f3": kF3 + bf16x3)
// Measured against the reference, all three give the same errors to within its own fp32
// rounding.
//
// The step has the BF16 path's structure (fast.cu):
//   GEMM-F   S = X_hat * W_subᵀ   (M = 256 batch rows / CTA pair, N = 256 classes, K = 512)
//            epilogue: P~ = exp(s*S - s) (fixed stabilizer, |cos| <= 1) -> HBM as bf16 hi / lo
//            planes (fp32, or hi / lo fp32 in the 3xTF32 mode), per-tile row sums and the label
//            logit (as fast.cu)
//   GEMM-dW  dW  = P~ᵀ * (diag(s*r) X_hat)     (M = 256 classes, K = B) -> fp32 rows
//   GEMM-dX  dX  = diag(s*r) * (P~ * W_sub)    (M = 256 batch, N = 512, K = M_w split) -> fp32
// with r_b = 1 / (B * sum_b); the one-hot part of G is applied exactly in fp32 by k_dx_reduce and
// the row update (LabelFix), as on the BF16 path.
//
// Shared-memory tiles (per CTA of a cta_group::2 pair; layouts per kind at their Cfg3):
//   kFm : tf32 rows (32 fp32 = 128 B, SW128) + the two bf16 planes (64-B rows, SW64), A and B
//   kDXb/kDWh: the BF16 path's layouts with 32 K per stage, hi | lo planes side by side
//   kF3 : A = X_hat rows / B = W_sub rows, K-major 128 rows x 32 fp32, hi + lo
//   kDX3: A = P~ rows K-major 16 fp32 (64B swizzle); B = W_sub MN-major 4 atoms of 32 d x 16 K
//   kDW3: A = P~ᵀ MN-major 4 atoms of 32 classes x 16 K rows; B = X_hat' as dX's B
// MN-major tf32 operands exist only in the 128B swizzle with 32-byte granules (UMMA layout type
// SWIZZLE_128B_BASE32B: 128 B along MN x 4 K rows per atom, granules XORed with row % 4), loaded
// by TMA with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B; LBO = stride between MN atoms, SBO = stride
// between 4-row K groups.
// Warp roles as fast.cu: warp 0 TMA producer, warp 1 MMA issuer (leader CTA), warp 2 TMEM
// allocator, warps 4-11 epilogue.
#include <cudaTypedefs.h>

#include "kernels.cuh"
#include "tc.cuh"

namespace xknn {

namespace {

enum Kind3 : int { kF3 = 0, kDX3 = 1, kDW3 = 2, kDXb = 3, kDWb = 4, kFm = 5, kDWh = 6 };
template <int KIND>
constexpr bool kIsF = KIND == kF3 || KIND == kFm;
template <int KIND>
constexpr bool kIsDX = KIND == kDX3 || KIND == kDXb;
template <int KIND>
constexpr bool kIsDW = KIND == kDW3 || KIND == kDWb || KIND == kDWh;

// Instruction descriptor, kind::tf32: TF32 A/B (format 2), fp32 D.
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t m, uint32_t n, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(0u)
      : "memory");
}

constexpr uint32_t kSwizzle128Base32 = 1;  // UMMA descriptor layout type

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct Gemm3Args {
  const SelState* st;
  uint32_t B, bpad, nbt, splits;
  float scale;
  const int32_t* label_col;
  float* p_hi;  // P~ [bpad][ldp] fp32 hi / lo (GEMM-F output)
  float* p_lo;
  __nv_bfloat16* pb_hi;  // ... or its two bf16 planes (bf16x3 backward GEMMs)
  __nv_bfloat16* pb_lo;
  uint64_t ldp;
  float* partial;    // F: [2 * class tiles][bpad] row sums; dX: split-K partial rows
  float* labelterm;  // F: [bpad]
};

template <int KIND>
struct Cfg3;
template <>
#ifndef XKNN_F3_KB
#define XKNN_F3_KB 32
#endif
struct Cfg3<kF3> {
  // KB fp32 of K per stage (KB * 4 B rows: 128B swizzle at 32, 64B at 16); 16 halves the stage
  // size for twice the stages -- more bytes in flight while the MMAs consume one
  static constexpr uint32_t KB = XKNN_F3_KB;
  static constexpr uint32_t STAGES = KB == 32 ? 3 : 6, A_BYTES = 2 * 128 * KB * 4,
                            B_BYTES = 2 * 128 * KB * 4;
  static constexpr uint32_t NBUF = 2, ACC = 256;
};
// GEMM-F in mixed precision: a*b ~ a_t*b_t + [bf16(a)*bf16(b - b_t) + bf16(a - a_t)*bf16(b)]
// with a_t = tf32(a): the leading product on kind::tf32, the two cross terms (each ~2^-11 of it)
// on kind::f16 at twice the rate -- 2 TF32-equivalents of MMA per product instead of 3.  A / B
// stage: the tf32 rows (32 fp32, 128 B, SW128) + the bf16 planes of a and of a - a_t (32 bf16,
// 64 B rows, SW64): the same 32 KB as the 3xTF32 hi / lo stage.
#ifndef XKNN_FM_KB
#define XKNN_FM_KB 32
#endif
template <>
struct Cfg3<kFm> {
  // KB = 16: half-size stages (64-B tf32 rows, SW64; 32-B bf16 rows, SW32), twice as many
  static constexpr uint32_t KB = XKNN_FM_KB, STAGES = KB == 32 ? 3 : 6,
                            A_BYTES = 128 * KB * 4 + 2 * 128 * KB * 2, B_BYTES = A_BYTES;
  static constexpr uint32_t TF = 128 * KB * 4, BP = 128 * KB * 2;  // tf32 rows, one bf16 plane
  static constexpr uint32_t NBUF = 2, ACC = 256;
};
template <>
struct Cfg3<kDX3> {
  static constexpr uint32_t STAGES = 4, A_BYTES = 2 * 128 * 64, B_BYTES = 2 * 8 * 2048;
  static constexpr uint32_t NBUF = 1, ACC = 512, KB = 16;
};
template <>
struct Cfg3<kDW3> {
  static constexpr uint32_t STAGES = 4, A_BYTES = 2 * 4 * 2048, B_BYTES = 2 * 8 * 2048;
  static constexpr uint32_t NBUF = 1, ACC = 512, KB = 16;
};
// bf16x3 backward GEMMs: P~, W_sub and X_hat' as two bf16 planes (hi = bf16(a), lo = bf16(a - hi),
// 16-17 significant bits) and a*b ~ lo*hi + hi*lo + hi*hi in kind::f16 -- the same three MMAs per
// product as 3xTF32 at twice the tensor-core rate, on the BF16 path's layouts (fast.cu) with 32
// K per stage.  KC = 32: A = 128 rows x 32 (dX: K-major, 64-B rows, SW64; dW: 2 MN-major atoms of
// 64 classes), B = 4 MN-major atoms of 64 d x 32 rows (SW128); hi | lo planes side by side.
template <>
struct Cfg3<kDXb> {
  static constexpr uint32_t STAGES = 4, A_BYTES = 2 * 128 * 32 * 2, B_BYTES = 2 * 4 * 4096;
  static constexpr uint32_t NBUF = 1, ACC = 512, KB = 32;
};
template <>
struct Cfg3<kDWb> {
  static constexpr uint32_t STAGES = 4, A_BYTES = 2 * 2 * 4096, B_BYTES = 2 * 4 * 4096;
  static constexpr uint32_t NBUF = 1, ACC = 512, KB = 32;
};
// kDWh: GEMM-dW bf16x3 in half-width units -- 256 classes x 256 d (one N = 256 instruction) --
// so that two 256-column accumulators fit TMEM and a unit's drain overlaps the next unit's MMAs
// (the K = B loop is short: at C2 a 512-wide unit's drain stalled the tensor core ~15 % of the
// time).  The two d-halves of a class tile are adjacent units (adjacent pairs, same time), so
// the second read of the P~ tile comes from L2.
#ifndef XKNN_DWH
#define XKNN_DWH 1
#endif
template <>
struct Cfg3<kDWh> {
  static constexpr uint32_t STAGES = 6, A_BYTES = 2 * 2 * 4096, B_BYTES = 2 * 2 * 4096;
  static constexpr uint32_t NBUF = 2, ACC = 256, KB = 32;
};
constexpr uint32_t kStg3 = 4096;  // per epilogue warp: one 32 x 32 fp32 staging block
#ifndef XKNN_PCONV
#define XKNN_PCONV 1
#endif
#ifndef XKNN_PCONV_TRUNC
#define XKNN_PCONV_TRUNC 0
#endif
#ifndef XKNN_PCONV_GROUPS
#define XKNN_PCONV_GROUPS 4
#endif
constexpr uint32_t kCvtGroups = XKNN_PCONV_GROUPS;
static_assert(4 % kCvtGroups == 0, "a converter group must own whole stages of the 4-stage ring");
// GEMM-dW / GEMM-dX read P~ as one fp32 array and split it hi/lo in shared memory (the epilogue
// warps, idle during the main loop, convert each stage before the MMA reads it) instead of
// reading HBM-resident hi and lo copies: P~ is written once (4 B per element, not 8) and each
// consumer reads half the bytes.  The split is the same round-to-nearest one, so the results are
// bit-identical.
template <int KIND>
constexpr bool kConv3 = XKNN_PCONV && (KIND == kDX3 || KIND == kDW3);

template <int KIND>
constexpr uint32_t smem_bytes3() {
  using C = Cfg3<KIND>;
  return C::STAGES * (C::A_BYTES + C::B_BYTES) + 8 * kStg3 + 1024 + 256;
}

struct Unit3 {
  uint32_t row0;    // F/dX: first batch row of the pair; dW: first class of the pair
  uint32_t t0, t1;  // F: class-tile range; dX: 16-class K-chunk range; dW: K-stage range
  uint32_t id;      // dX: partial slot; dW: partial slot of a split tail unit
  bool valid;
  bool part;        // dW: a K-partial of a tail unit (dw_split)
};

template <int KIND>
__device__ __forceinline__ uint32_t num_units3(const Gemm3Args& a, uint32_t mw) {
  if (KIND == kDWh) return 2 * ((mw + 255) / 256);
  if (kIsDW<KIND>) {
    const uint32_t units = (mw + 255) / 256;
    const DwSplit sp = dw_split(units, gridDim.x / 2);
    return sp.full + (units - sp.full) * sp.s;
  }
  return a.nbt * a.splits;
}

template <int KIND>
__device__ __forceinline__ Unit3 unit3_of(const Gemm3Args& a, uint32_t mw, uint32_t u) {
  Unit3 x{};
  x.id = u;
  if (KIND == kDWh) {  // class tile u / 2, d-half u % 2 (in id)
    x.valid = true;
    x.row0 = (u >> 1) * 256;
    x.t0 = 0;
    x.t1 = a.bpad / Cfg3<KIND>::KB;
    x.id = u & 1;
    return x;
  }
  if (kIsDW<KIND>) {
    const uint32_t nk = a.bpad / Cfg3<KIND>::KB;
    const DwSplit sp = dw_split((mw + 255) / 256, gridDim.x / 2);
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
    x.id = v;
    x.part = true;
    return x;
  }
  const uint32_t bp = u % a.nbt, r = u / a.nbt;
  const uint32_t nt = kIsF<KIND> ? (mw + 255) / 256 : (mw + Cfg3<KIND>::KB - 1) / Cfg3<KIND>::KB;
  x.row0 = bp * 256;
  x.t0 = (uint32_t)((uint64_t)r * nt / a.splits);
  x.t1 = (uint32_t)((uint64_t)(r + 1) * nt / a.splits);
  x.valid = kIsDX<KIND> || x.t1 > x.t0;  // dX units always write their (maybe zero) partial
  return x;
}

// one thread's 32 fp32 of a row into a 128B-swizzled 32 x 32 staging block (TMA-store layout)
__device__ __forceinline__ void stage_f32(uint8_t* buf, uint32_t r, const float (&v)[32]) {
#pragma unroll
  for (uint32_t c = 0; c < 8; ++c) {
    float4* d = reinterpret_cast<float4*>(buf + r * 128 + ((c ^ (r & 7)) * 16));
    *d = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
}
// the same for the tf32 split of the values: LO = false: tf32(v), LO = true: v - tf32(v)
template <bool LO>
__device__ __forceinline__ void stage_split(uint8_t* buf, uint32_t r, const float (&v)[32]) {
#pragma unroll
  for (uint32_t c = 0; c < 8; ++c) {
    float t[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float x = v[4 * c + i], hi = tf32_rna(x);
      t[i] = LO ? x - hi : hi;
    }
    float4* d = reinterpret_cast<float4*>(buf + r * 128 + ((c ^ (r & 7)) * 16));
    *d = make_float4(t[0], t[1], t[2], t[3]);
  }
}
// ... and the block to global rows `ld` floats apart: lane l writes row 4i + l/8, 16-B unit l%8
// (four full 128-B row segments per instruction)
__device__ __forceinline__ void store_f32_block(const uint8_t* buf, float* dst, uint64_t ld,
                                                uint32_t lane) {
  const uint32_t c = lane & 7;
#pragma unroll
  for (uint32_t i = 0; i < 8; ++i) {
    const uint32_t r = 4 * i + (lane >> 3);
    const float4 v = *reinterpret_cast<const float4*>(buf + r * 128 + ((c ^ (r & 7)) * 16));
    *reinterpret_cast<float4*>(dst + (uint64_t)r * ld + c * 4) = v;
  }
  __syncwarp();
}

// bf16 planes of a pair of values: hi = bf16(v), lo = bf16(v - hi) (v - hi is exact)
__device__ __forceinline__ void split_bf16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(a - hf.x, b - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
// one thread's 32 values as bf16 hi / lo planes into two 32 x 64 B staging blocks (buf, buf +
// 2 KB), 16-B unit c of row r at c ^ ((r >> 1) & 3) (conflict-free both ways)
__device__ __forceinline__ void stage_bf16_planes(uint8_t* buf, uint32_t r, const float (&v)[32]) {
#pragma unroll
  for (uint32_t c = 0; c < 4; ++c) {
    uint4 h, l;
    split_bf16x2(v[8 * c + 0], v[8 * c + 1], h.x, l.x);
    split_bf16x2(v[8 * c + 2], v[8 * c + 3], h.y, l.y);
    split_bf16x2(v[8 * c + 4], v[8 * c + 5], h.z, l.z);
    split_bf16x2(v[8 * c + 6], v[8 * c + 7], h.w, l.w);
    const uint32_t off = r * 64 + ((c ^ ((r >> 1) & 3)) * 16);
    *reinterpret_cast<uint4*>(buf + off) = h;
    *reinterpret_cast<uint4*>(buf + 2048 + off) = l;
  }
}
// ... and both blocks to global rows `ld` elements apart: lane l writes row 8i + l/4, 16-B unit
// l%4 (eight full 64-B row segments per instruction and plane)
__device__ __forceinline__ void store_bf16_planes(const uint8_t* buf, __nv_bfloat16* dhi,
                                                  __nv_bfloat16* dlo, uint64_t ld, uint32_t lane) {
  const uint32_t c = lane & 3;
#pragma unroll
  for (uint32_t i = 0; i < 4; ++i) {
    const uint32_t r = 8 * i + (lane >> 2), off = r * 64 + ((c ^ ((r >> 1) & 3)) * 16);
    *reinterpret_cast<uint4*>(dhi + (uint64_t)r * ld + c * 8) =
        *reinterpret_cast<const uint4*>(buf + off);
    *reinterpret_cast<uint4*>(dlo + (uint64_t)r * ld + c * 8) =
        *reinterpret_cast<const uint4*>(buf + 2048 + off);
  }
  __syncwarp();
}

template <int KIND>
__global__ void __launch_bounds__(384, 1)
    k_gemm3(const __grid_constant__ CUtensorMap tmAhi, const __grid_constant__ CUtensorMap tmAlo,
            const __grid_constant__ CUtensorMap tmBhi, const __grid_constant__ CUtensorMap tmBlo,
            const __grid_constant__ CUtensorMap tmOut, const __grid_constant__ CUtensorMap tmOut2,
            const __grid_constant__ CUtensorMap tmAd, const __grid_constant__ CUtensorMap tmBd,
            Gemm3Args a) {
  using C = Cfg3<KIND>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (uint32_t)(reinterpret_cast<uintptr_t>(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                // [stage][hi | lo]
  uint8_t* sB = sA + C::STAGES * C::A_BYTES;         // [stage][hi | lo]
  uint8_t* sStg = sB + C::STAGES * C::B_BYTES;       // epilogue staging, 8 warps x 4 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStg + 8 * kStg3);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* lfull = tempty + 2;          // kConv3: this CTA's stage bytes landed (local TMA)
  uint64_t* conv = lfull + C::STAGES;    // kConv3 (leader): both CTAs' A stage split hi/lo
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(conv + C::STAGES);
  constexpr bool CONV = kConv3<KIND>;
  constexpr bool BF = KIND == kDXb || KIND == kDWb || KIND == kDWh;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = tc::cluster_ctarank() & 1;
  const bool leader = cta == 0;
  const uint32_t pair = blockIdx.x / 2, npairs = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    for (uint32_t s = 0; s < C::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
      tc::mbar_init(&lfull[s], 1);
      tc::mbar_init(&conv[s], 2 * (8 / kCvtGroups));  // one group's warps in each CTA
    }
    for (uint32_t s = 0; s < 2; ++s) {
      tc::mbar_init(&tfull[s], 1);
      tc::mbar_init(&tempty[s], 16);  // 8 epilogue warps in each CTA of the pair
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmAhi);
    tc::tma_prefetch(&tmAlo);
    tc::tma_prefetch(&tmBhi);
    tc::tma_prefetch(&tmBlo);
    if (KIND == kFm) {
      tc::tma_prefetch(&tmAd);
      tc::tma_prefetch(&tmBd);
    }
    if (!kIsF<KIND>) tc::tma_prefetch(&tmOut);
  }
  if (warp == 2) tc::tmem_alloc_2sm<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;
  griddep_wait();

  const uint32_t mw = a.st->active_count;
  const uint32_t nunits = num_units3<KIND>(a, mw);

  if (warp == 0) {
    // ================= TMA producer (both CTAs load their half) =================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (uint32_t u = pair; u < nunits; u += npairs) {
        const Unit3 x = unit3_of<KIND>(a, mw, u);
        if (!x.valid) continue;
        const int32_t myrow = (int32_t)(x.row0 + cta * 128);
        const uint32_t nk = kIsF<KIND> ? (x.t1 - x.t0) * (512 / C::KB) : x.t1 - x.t0;
        for (uint32_t k = 0; k < nk; ++k) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          if (CONV)  // this CTA's fp32 A (the hi half of the A stage) and hi/lo B
            tc::mbar_expect_tx(&lfull[stage], C::A_BYTES / 2 + C::B_BYTES);
          else if (leader)
            tc::mbar_expect_tx(&full[stage], 2 * (C::A_BYTES + C::B_BYTES));
          // CONV: loads complete on this CTA's own barrier (the converters wait on it)
          auto load = [&](void* dst, const CUtensorMap* m, int32_t c0, int32_t c1) {
            if (CONV)
              tc::tma_load_2d(dst, m, &lfull[stage], c0, c1);
            else
              tc::tma_load_2d_2sm(dst, m, &full[stage], c0, c1);
          };
          uint8_t* dA = sA + stage * C::A_BYTES;
          uint8_t* dB = sB + stage * C::B_BYTES;
          if (kIsF<KIND>) {
            constexpr uint32_t NKB = 512 / C::KB;  // stages per class tile
            const int32_t kc = (int32_t)((k % NKB) * C::KB);
            const int32_t crow = (int32_t)((x.t0 + k / NKB) * 256 + cta * 128);
            if (KIND == kFm) {  // tf32 rows | bf16(a) | bf16(a - a_t)
              constexpr uint32_t TF = Cfg3<kFm>::TF, BP = Cfg3<kFm>::BP;
              tc::tma_load_2d_2sm(dA, &tmAhi, &full[stage], kc, myrow);
              tc::tma_load_2d_2sm(dA + TF, &tmAlo, &full[stage], kc, myrow);
              tc::tma_load_2d_2sm(dA + TF + BP, &tmAd, &full[stage], kc, myrow);
              tc::tma_load_2d_2sm(dB, &tmBhi, &full[stage], kc, crow);
              tc::tma_load_2d_2sm(dB + TF, &tmBlo, &full[stage], kc, crow);
              tc::tma_load_2d_2sm(dB + TF + BP, &tmBd, &full[stage], kc, crow);
            } else {
              tc::tma_load_2d_2sm(dA, &tmAhi, &full[stage], kc, myrow);
              tc::tma_load_2d_2sm(dA + C::A_BYTES / 2, &tmAlo, &full[stage], kc, myrow);
              tc::tma_load_2d_2sm(dB, &tmBhi, &full[stage], kc, crow);
              tc::tma_load_2d_2sm(dB + C::B_BYTES / 2, &tmBlo, &full[stage], kc, crow);
            }
          } else if (BF) {
            const int32_t kk = (int32_t)((x.t0 + k) * 32);
            if (kIsDX<KIND>) {  // P~ planes [b][class]: this CTA's 128 batch rows, 32 classes
              load(dA, &tmAhi, kk, myrow);
              load(dA + C::A_BYTES / 2, &tmAlo, kk, myrow);
            } else {  // P~ᵀ planes: this CTA's 128 classes (2 atoms of 64) at batch rows kk..+31
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                load(dA + j * 4096, &tmAhi, myrow + 64 * j, kk);
                load(dA + C::A_BYTES / 2 + j * 4096, &tmAlo, myrow + 64 * j, kk);
              }
            }
            // B planes [K rows][512 d]: this CTA's 128 d of each 256-wide N instruction j (kDWh:
            // only the unit's d-half)
#pragma unroll
            for (int j = 0; j < (KIND == kDWh ? 1 : 2); ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int32_t dc = (int32_t)(256 * (KIND == kDWh ? x.id : j) + 128 * cta + 64 * h);
                load(dB + (j * 2 + h) * 4096, &tmBhi, dc, kk);
                load(dB + C::B_BYTES / 2 + (j * 2 + h) * 4096, &tmBlo, dc, kk);
              }
          } else {
            const int32_t kk = (int32_t)((x.t0 + k) * 16);
            if (KIND == kDX3) {  // P~ [b][class]: this CTA's 128 batch rows, 16 classes
              load(dA, &tmAhi, kk, myrow);
              if (!CONV) load(dA + C::A_BYTES / 2, &tmAlo, kk, myrow);
            } else {  // P~ᵀ: this CTA's 128 classes (4 atoms of 32) at batch rows kk..kk+15
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                load(dA + t * 2048, &tmAhi, myrow + 32 * t, kk);
                if (!CONV) load(dA + C::A_BYTES / 2 + t * 2048, &tmAlo, myrow + 32 * t, kk);
              }
            }
            // B [K rows][512 d]: this CTA's 128 d of each 256-wide N instruction j, 4 atoms
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const int32_t dc = (int32_t)(256 * j + 128 * cta + 32 * t);
                load(dB + (j * 4 + t) * 2048, &tmBhi, dc, kk);
                load(dB + C::B_BYTES / 2 + (j * 4 + t) * 2048, &tmBlo, dc, kk);
              }
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA, one thread) =================
    if (leader && lane == 0) {
      uint32_t stage = 0, phase = 0, buf = 0, tphase = 0;
      for (uint32_t u = pair; u < nunits; u += npairs) {
        const Unit3 x = unit3_of<KIND>(a, mw, u);
        if (!x.valid) continue;
        const uint32_t ntile = kIsF<KIND> ? x.t1 - x.t0 : 1;
        for (uint32_t t = 0; t < ntile; ++t) {
          tc::mbar_wait(&tempty[buf], tphase ^ 1);
          tc::fence_after_sync();
          const uint32_t dcol = tbase + buf * C::ACC;
          const uint32_t nk = kIsF<KIND> ? 512 / C::KB : x.t1 - x.t0;
          for (uint32_t k = 0; k < nk; ++k) {
            if (CONV)
              tc::mbar_wait_cluster(&conv[stage], phase);
            else
              tc::mbar_wait(&full[stage], phase);
            tc::fence_after_sync();
            const uint32_t ah = tc::smem_u32(sA + stage * C::A_BYTES), al = ah + C::A_BYTES / 2;
            const uint32_t bh = tc::smem_u32(sB + stage * C::B_BYTES), bl = bh + C::B_BYTES / 2;
            if (KIND == kFm) {
              constexpr uint32_t idt = idesc_tf32(256, 256, false, false);
              constexpr uint32_t idb = tc::idesc_bf16(256, 256, false, false);
              constexpr uint32_t KB = Cfg3<kFm>::KB, TF = Cfg3<kFm>::TF, BP = Cfg3<kFm>::BP;
              // tf32 rows of KB * 4 B, bf16 rows of KB * 2 B: 8-row groups, matching swizzles
              constexpr uint32_t SWT = KB == 32 ? tc::kSwizzle128 : tc::kSwizzle64;
              constexpr uint32_t SWB = KB == 32 ? tc::kSwizzle64 : tc::kSwizzle32;
#pragma unroll
              for (uint32_t kk = 0; kk < KB / 16; ++kk) {  // cross terms first: K = 16 bf16 = 32 B
                const uint64_t dah = tc::smem_desc(ah + TF + kk * 32, 16, KB * 16, SWB);
                const uint64_t dad = tc::smem_desc(ah + TF + BP + kk * 32, 16, KB * 16, SWB);
                const uint64_t dbh = tc::smem_desc(bh + TF + kk * 32, 16, KB * 16, SWB);
                const uint64_t dbd = tc::smem_desc(bh + TF + BP + kk * 32, 16, KB * 16, SWB);
                tc::mma_bf16_2sm(dcol, dah, dbd, idb, (k | kk) != 0);
                tc::mma_bf16_2sm(dcol, dad, dbh, idb, 1u);
              }
#pragma unroll
              for (uint32_t kk = 0; kk < KB / 8; ++kk)  // the tf32 products: K = 8 fp32 = 32 B
                mma_tf32_2sm(dcol, tc::smem_desc(ah + kk * 32, 16, KB * 32, SWT),
                             tc::smem_desc(bh + kk * 32, 16, KB * 32, SWT), idt, 1u);
            } else if (KIND == kF3) {
              constexpr uint32_t id = idesc_tf32(256, 256, false, false);
              constexpr uint32_t SBO = C::KB * 4 * 8;  // 8-row group of KB * 4-byte rows
              constexpr uint32_t SW = C::KB == 32 ? tc::kSwizzle128 : tc::kSwizzle64;
#pragma unroll
              for (uint32_t kk = 0; kk < C::KB / 8; ++kk) {  // K = 8 fp32 = 32 B per instruction
                const uint64_t dah = tc::smem_desc(ah + kk * 32, 16, SBO, SW);
                const uint64_t dal = tc::smem_desc(al + kk * 32, 16, SBO, SW);
                const uint64_t dbh = tc::smem_desc(bh + kk * 32, 16, SBO, SW);
                const uint64_t dbl = tc::smem_desc(bl + kk * 32, 16, SBO, SW);
                mma_tf32_2sm(dcol, dal, dbh, id, (k | kk) != 0);  // small terms first
                mma_tf32_2sm(dcol, dah, dbl, id, 1u);
                mma_tf32_2sm(dcol, dah, dbh, id, 1u);
              }
            } else if (BF) {
              constexpr uint32_t id = tc::idesc_bf16(256, 256, kIsDW<KIND>, true);
#pragma unroll
              for (uint32_t kk = 0; kk < 2; ++kk) {  // K = 16 per instruction
                const uint64_t dah =
                    kIsDX<KIND> ? tc::smem_desc(ah + kk * 32, 16, 512, tc::kSwizzle64)
                                : tc::smem_desc(ah + kk * 2048, 4096, 1024, tc::kSwizzle128);
                const uint64_t dal =
                    kIsDX<KIND> ? tc::smem_desc(al + kk * 32, 16, 512, tc::kSwizzle64)
                                : tc::smem_desc(al + kk * 2048, 4096, 1024, tc::kSwizzle128);
#pragma unroll
                for (uint32_t j = 0; j < (KIND == kDWh ? 1u : 2u); ++j) {
                  const uint64_t dbh =
                      tc::smem_desc(bh + j * 8192 + kk * 2048, 4096, 1024, tc::kSwizzle128);
                  const uint64_t dbl =
                      tc::smem_desc(bl + j * 8192 + kk * 2048, 4096, 1024, tc::kSwizzle128);
                  tc::mma_bf16_2sm(dcol + j * 256, dal, dbh, id, (k | kk) != 0);
                  tc::mma_bf16_2sm(dcol + j * 256, dah, dbl, id, 1u);
                  tc::mma_bf16_2sm(dcol + j * 256, dah, dbh, id, 1u);
                }
              }
            } else {
              constexpr uint32_t id = idesc_tf32(256, 256, KIND == kDW3, true);
#pragma unroll
              for (uint32_t ks = 0; ks < 2; ++ks) {  // K = 8 rows per instruction
                const uint64_t dah =
                    KIND == kDX3 ? tc::smem_desc(ah + ks * 32, 16, 512, tc::kSwizzle64)
                                 : tc::smem_desc(ah + ks * 1024, 2048, 512, kSwizzle128Base32);
                const uint64_t dal =
                    KIND == kDX3 ? tc::smem_desc(al + ks * 32, 16, 512, tc::kSwizzle64)
                                 : tc::smem_desc(al + ks * 1024, 2048, 512, kSwizzle128Base32);
#pragma unroll
                for (uint32_t j = 0; j < 2; ++j) {
                  const uint64_t dbh =
                      tc::smem_desc(bh + j * 8192 + ks * 1024, 2048, 512, kSwizzle128Base32);
                  const uint64_t dbl =
                      tc::smem_desc(bl + j * 8192 + ks * 1024, 2048, 512, kSwizzle128Base32);
                  mma_tf32_2sm(dcol + j * 256, dal, dbh, id, (k | ks) != 0);
                  mma_tf32_2sm(dcol + j * 256, dah, dbl, id, 1u);
                  mma_tf32_2sm(dcol + j * 256, dah, dbh, id, 1u);
                }
              }
            }
            tc::mma_commit_2sm(&empty[stage]);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
          if (nk) {
            tc::mma_commit_2sm(&tfull[buf]);
          } else {  // an empty split-K range: the epilogue writes zeros
            tc::mbar_arrive_remote(&tfull[buf], 0);
            tc::mbar_arrive_remote(&tfull[buf], 1);
          }
          if (++buf == C::NBUF) { buf = 0; tphase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue (both CTAs: their own 128 rows) =================
    const uint32_t q = warp & 3, h = (warp - 4) >> 2, ew = warp - 4;
    const uint32_t row = q * 32 + lane;
    const uint32_t lane_addr = (q * 32) << 16;
    uint8_t* stg = sStg + ew * kStg3;
    uint32_t buf = 0, tphase = 0;
    // CONV: the A stages in MMA order, split hi/lo in place: hi = tf32(x) over x, lo = x - hi
    // into the stage's second half (both halves keep the TMA swizzle, the split is elementwise)
    // The warps form kCvtGroups groups that take the stages in turn, so that one stage's
    // wait -> split -> proxy fence -> arrive chain overlaps the next stage's.
    constexpr uint32_t NG = kCvtGroups, GT = 256 / NG;  // groups, threads per group
    const uint32_t grp = ew / (8 / NG), et = (ew % (8 / NG)) * 32 + lane;
    uint32_t cdone = 0, cend = 0;
    auto convert_to = [&](uint32_t target) {
      for (; cdone < target; ++cdone) {
        if (cdone % NG != grp) continue;
        const uint32_t cstage = cdone % C::STAGES, cphase = (cdone / C::STAGES) & 1;
        tc::mbar_wait(&lfull[cstage], cphase);
        float4* ph = reinterpret_cast<float4*>(sA + cstage * C::A_BYTES);
        float4* pl = reinterpret_cast<float4*>(sA + cstage * C::A_BYTES + C::A_BYTES / 2);
#pragma unroll
        for (uint32_t i = 0; i < C::A_BYTES / 2 / 16 / GT; ++i) {
          const float4 v = ph[et + GT * i];
#if XKNN_PCONV_TRUNC
          auto tr = [](float f) { return __uint_as_float(__float_as_uint(f) & 0xffffe000u); };
          const float4 hi = make_float4(tr(v.x), tr(v.y), tr(v.z), tr(v.w));
#else
          const float4 hi = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
          ph[et + GT * i] = hi;
#endif
          pl[et + GT * i] = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
        }
        tc::fence_proxy_async_smem();  // generic-proxy writes -> the tensor core's reads
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_remote(&conv[cstage], 0);
      }
    };
    for (uint32_t u = pair; u < nunits; u += npairs) {
      const Unit3 x = unit3_of<KIND>(a, mw, u);
      if (!x.valid) continue;
      if (CONV) {
        // this unit's stages, then the next unit's first ones (already loadable: the MMA has
        // released every stage once this unit's last one is converted), so that its MMA can
        // start as soon as the accumulator below is drained
        cend += x.t1 - x.t0;
        uint32_t pre = 0;
        if (u + npairs < nunits) {
          const Unit3 y = unit3_of<KIND>(a, mw, u + npairs);
          pre = min(C::STAGES, y.t1 - y.t0);
        }
        convert_to(cend + pre);
      }
      const uint32_t ntile = kIsF<KIND> ? x.t1 - x.t0 : 1;
      for (uint32_t t = 0; t < ntile; ++t) {
        tc::mbar_wait(&tfull[buf], tphase);
        tc::fence_after_sync();
        const uint32_t tb = tbase + buf * C::ACC + lane_addr;
        const int32_t grow0 = (int32_t)(x.row0 + cta * 128 + q * 32);  // this warp's 32 rows
        if (kIsF<KIND>) {
          const uint32_t ct = x.t0 + t;
          const uint32_t b = x.row0 + cta * 128 + row;
          const bool vrow = b < a.B;
          const int32_t lc = vrow ? a.label_col[b] : -1;
          const float k2 = a.scale * 1.4426950408889634f;
          float sum = 0.f, lab = 0.f;
          bool has = false;
          auto process = [&](const uint32_t (&r)[32], uint32_t ch) {
            const uint32_t c0 = ct * 256 + h * 128 + ch * 32;
            float e[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const bool ok = vrow && c0 + j < mw;
              e[j] = ok ? ex2_approx(fmaf(__uint_as_float(r[j]), k2, -k2)) : 0.f;
              sum += e[j];
            }
            if (lc >= (int32_t)c0 && lc < (int32_t)c0 + 32) {  // at most once per row
              const int32_t idx = lc - (int32_t)c0;
              float sel = 0.f;
#pragma unroll
              for (int j = 0; j < 32; ++j) sel = (j == idx) ? __uint_as_float(r[j]) : sel;
              lab = sel * a.scale;
              has = true;
            }
            const uint64_t off = (uint64_t)grow0 * a.ldp + c0;
            if (a.pb_hi) {  // bf16 hi / lo planes for the bf16x3 backward GEMMs
              stage_bf16_planes(stg, lane, e);
              __syncwarp();
              store_bf16_planes(stg, a.pb_hi + off, a.pb_lo + off, a.ldp, lane);
            } else if (XKNN_PCONV) {  // one fp32 P~: its consumers split it in shared memory
              stage_f32(stg, lane, e);
              __syncwarp();
              store_f32_block(stg, a.p_hi + off, a.ldp, lane);
            } else {
              stage_split<false>(stg, lane, e);
              __syncwarp();
              store_f32_block(stg, a.p_hi + off, a.ldp, lane);
              stage_split<true>(stg, lane, e);
              __syncwarp();
              store_f32_block(stg, a.p_lo + off, a.ldp, lane);
            }
          };
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
          if (lane == 0) tc::mbar_arrive_remote_relaxed(&tempty[buf], 0);
          process(rb, 3);
          a.partial[(uint64_t)(ct * 2 + h) * a.bpad + b] = sum;
          if (has) a.labelterm[b] = lab - a.scale;
        } else {
          // dX: split-K partial rows of unit x.id; dW: fp32 dW rows (compact active order), or
          // the K-partial rows of a split tail unit (slot x.id, through tmOut2)
          const bool part = kIsDW<KIND> && x.part;
          const int32_t orow = (kIsDX<KIND> || part) ? (int32_t)(x.id * 256) + grow0 - (int32_t)x.row0
                                                      : grow0;
          const bool zero = kIsDX<KIND> && x.t1 == x.t0;
#pragma unroll 1
          for (uint32_t ch = 0; ch < C::ACC / 64; ++ch) {
            const uint32_t col = h * (C::ACC / 2) + ch * 32;
            float v[32];
            if (!zero) {
              tc::tmem_ld32(tb + col, v);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = 0.f;
            }
            stage_f32(stg, lane, v);
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tc::tma_store_2d(part ? &tmOut2 : &tmOut, stg,
                               (int32_t)(col + (KIND == kDWh ? x.id * 256 : 0)), orow);
              tc::tma_store_commit();
              tc::tma_store_wait_read<0>();
            }
            __syncwarp();
          }
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_remote_relaxed(&tempty[buf], 0);
        }
        if (++buf == C::NBUF) { buf = 0; tphase ^= 1; }
      }
    }
    if (lane == 0) tc::tma_store_wait_all();
    __syncwarp();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();
  if (warp == 2) {
    tc::fence_after_sync();
    tc::tmem_dealloc_2sm<512>(tbase);
  }
}

// X_hat' = x_hat * s / (B * sum) split hi/lo (pad rows zero); the batch rows of every local label
// column linked into lists for the row update; the step's loss (block 0, k_loss's arithmetic)
__global__ void k_fixup32(const double* __restrict__ red, const int32_t* __restrict__ lcol,
                          const float* __restrict__ X, const float* __restrict__ xnorm, uint32_t B,
                          uint32_t bpad, float scale, int32_t* __restrict__ lab_head,
                          int32_t* __restrict__ lab_next, float* __restrict__ xs_hi,
                          float* __restrict__ xs_lo, __nv_bfloat16* __restrict__ xsb_hi,
                          __nv_bfloat16* __restrict__ xsb_lo, double* __restrict__ loss,
                          SelState* st, unsigned long long* err) {
  griddep_wait();
  griddep_launch();
  if (blockIdx.x == 0) {
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
    float4* dh = reinterpret_cast<float4*>(xs_hi + (uint64_t)b * 512);
    float4* dl = reinterpret_cast<float4*>(xs_lo + (uint64_t)b * 512);
    uint2* bh = reinterpret_cast<uint2*>(xsb_hi + (uint64_t)b * 512);
    uint2* bl = reinterpret_cast<uint2*>(xsb_lo + (uint64_t)b * 512);
    if (b >= B) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (xsb_hi) {
          bh[lane + 32 * c] = make_uint2(0u, 0u);
          bl[lane + 32 * c] = make_uint2(0u, 0u);
        } else {
          dh[lane + 32 * c] = make_float4(0.f, 0.f, 0.f, 0.f);
          dl[lane + 32 * c] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      continue;
    }
    const int32_t lc = lcol[b];
    if (lane == 0 && lc >= 0) lab_next[b] = atomicExch(&lab_head[lc], (int32_t)b);
    const float inv = 1.0f / xnorm[b];
    const float rs = (float)((double)scale / ((double)B * red[b]));
    const float4* xp = reinterpret_cast<const float4*>(X + (uint64_t)b * 512);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float4 x = xp[lane + 32 * c];
      const float4 v = make_float4(__fmul_rn(__fmul_rn(x.x, inv), rs), __fmul_rn(__fmul_rn(x.y, inv), rs),
                                   __fmul_rn(__fmul_rn(x.z, inv), rs), __fmul_rn(__fmul_rn(x.w, inv), rs));
      if (xsb_hi) {  // bf16 planes (bf16x3 GEMM-dW)
        uint2 h, l;
        split_bf16x2(v.x, v.y, h.x, l.x);
        split_bf16x2(v.z, v.w, h.y, l.y);
        bh[lane + 32 * c] = h;
        bl[lane + 32 * c] = l;
        continue;
      }
      const float4 hi = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
      dh[lane + 32 * c] = hi;
      dl[lane + 32 * c] = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
    }
  }
}

// rows [count, round_up(count, 256)) of W_sub hi/lo must be zero for GEMM-dX's K loop
__global__ void k_zero_rows32(const SelState* st, float* whi, float* wlo, __nv_bfloat16* wbh,
                              __nv_bfloat16* wbl, uint32_t cap_rows) {
  griddep_wait();
  griddep_launch();
  const uint32_t c = st->active_count;
  const uint32_t e = min(cap_rows, (c + 255) / 256 * 256);
  const uint64_t n = (uint64_t)(e - c) * 512 / 4;
  float4* ph = reinterpret_cast<float4*>(whi + (uint64_t)c * 512);
  float4* pl = wlo ? reinterpret_cast<float4*>(wlo + (uint64_t)c * 512) : nullptr;
  uint2* bh = wbh ? reinterpret_cast<uint2*>(wbh + (uint64_t)c * 512) : nullptr;
  uint2* bl = wbh ? reinterpret_cast<uint2*>(wbl + (uint64_t)c * 512) : nullptr;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    ph[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (pl) pl[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (bh) {
      bh[i] = make_uint2(0u, 0u);
      bl[i] = make_uint2(0u, 0u);
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn3() {
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

// fp32 (or bf16) row-major [outer][inner] tensor, box_inner x box_outer
bool make_map32(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw, bool bf16 = false) {
  auto fn = encode_fn3();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * (bf16 ? 2 : 4)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
            const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

struct Fast32State {
  uint32_t bpad = 0, mwpad = 0;
  uint64_t dx_units_cap = 0;
  float *xh_hi = nullptr, *xh_lo = nullptr;  // X_hat hi/lo [bpad][512]
  float *xs_hi = nullptr, *xs_lo = nullptr;  // X_hat' hi/lo [bpad][512]
  float *w_hi = nullptr, *w_lo = nullptr;    // W_sub hi/lo [mwpad][512]
  float *p_hi = nullptr, *p_lo = nullptr;    // P~ [bpad][mwpad] (fp32; hi/lo if !XKNN_PCONV)
  float* partial_f = nullptr;                // [2 * mwpad/256][bpad]
  float* labelterm = nullptr;                // [bpad]
  float* partial_dx = nullptr;               // [units][256][512]
  float* dW32 = nullptr;                     // [mwpad][512]
  float* dw_part = nullptr;                  // [74 slots][256][512] tail-unit K-partials
  int32_t* lab_head = nullptr;               // [mwpad]
  int32_t* lab_next = nullptr;               // [bpad]
  CUtensorMap mF_Ah, mF_Al, mF_Bh, mF_Bl;    // X_hat, W_sub (K-major, 32 x 128 boxes)
  CUtensorMap mDX_Ah, mDX_Al, mDX_Bh, mDX_Bl, mDX_st;  // P~ (16 x 128, SW64), W_sub (32 x 16)
  CUtensorMap mDW_Ah, mDW_Al, mDW_Bh, mDW_Bl, mDW_st;  // P~ (32 x 16), X_hat' (32 x 16)
  CUtensorMap mDWP_st;                                 // dW tail-unit K-partials
  // GEMM arithmetic (XKNN_FP32_GEMM): "mixed" (default) = GEMM-F mixed tf32/bf16 + bf16x3
  // GEMM-dW/dX; "f3" = 3xTF32 GEMM-F + bf16x3 dW/dX; "3xtf32" = 3xTF32 throughout.  The bf16
  // planes of P~, W_sub and X_hat' replace P~ fp32 and X_hat' hi/lo as the bf16x3 operands.
  bool bfb = true, mixed = true;
  __nv_bfloat16 *xb_hi = nullptr, *xd = nullptr;  // mixed GEMM-F: bf16(x_hat), bf16(x_hat - tf32)
  __nv_bfloat16* wd = nullptr;                      // ... bf16(w_sub - tf32(w_sub)) [mwpad][512]
  CUtensorMap mF_Ad, mF_Bd;
  __nv_bfloat16 *pb_hi = nullptr, *pb_lo = nullptr;    // P~ [bpad][mwpad]
  __nv_bfloat16 *wb_hi = nullptr, *wb_lo = nullptr;    // W_sub [mwpad][512]
  __nv_bfloat16 *xsb_hi = nullptr, *xsb_lo = nullptr;  // X_hat' [bpad][512]
};

xknn_status_t Layer::init_fast32() {
  auto* f = new Fast32State;
  fast32 = f;
  if (d != 512) return fail_msg(XKNN_ERR_UNSUPPORTED, "FP32 tensor-core path is specialised for D = 512");
  f->bpad = (uint32_t)((bmax + 255) / 256 * 256);
  f->mwpad = (uint32_t)((mw_cap + 255) / 256 * 256);
  ldp = f->mwpad;
  if (const char* e = getenv("XKNN_FP32_GEMM")) {
    if (strcmp(e, "mixed") && strcmp(e, "f3") && strcmp(e, "3xtf32"))
      return fail_msg(XKNN_ERR_CONFIG, "XKNN_FP32_GEMM must be mixed, f3 or 3xtf32");
    f->mixed = strcmp(e, "mixed") == 0;
    f->bfb = strcmp(e, "3xtf32") != 0;
  }
  const uint64_t xb = (uint64_t)f->bpad * 512, wb = (uint64_t)f->mwpad * 512,
                 pb = (uint64_t)f->bpad * f->mwpad;
  for (float** p : {&f->xh_hi, &f->xh_lo, &f->xs_hi, &f->xs_lo}) {
    XK_CUDA(dalloc(p, xb));
    XK_CUDA(cudaMemsetAsync(*p, 0, xb * 4, stream));
  }
  for (float** p : {&f->w_hi, &f->w_lo}) {
    if (f->mixed && p == &f->w_lo) continue;
    XK_CUDA(dalloc(p, wb));
    XK_CUDA(cudaMemsetAsync(*p, 0, wb * 4, stream));
  }
  if (f->mixed) {
    for (auto* p : {&f->xb_hi, &f->xd}) {
      XK_CUDA(dalloc(p, xb));
      XK_CUDA(cudaMemsetAsync(*p, 0, xb * 2, stream));
    }
    XK_CUDA(dalloc(&f->wd, wb));
    XK_CUDA(cudaMemsetAsync(f->wd, 0, wb * 2, stream));
  }
  if (f->bfb) {
    for (auto* p : {&f->pb_hi, &f->pb_lo}) {
      XK_CUDA(dalloc(p, pb));
      XK_CUDA(cudaMemsetAsync(*p, 0, pb * 2, stream));
    }
    for (auto* p : {&f->wb_hi, &f->wb_lo}) {
      XK_CUDA(dalloc(p, wb));
      XK_CUDA(cudaMemsetAsync(*p, 0, wb * 2, stream));
    }
    for (auto* p : {&f->xsb_hi, &f->xsb_lo}) {
      XK_CUDA(dalloc(p, xb));
      XK_CUDA(cudaMemsetAsync(*p, 0, xb * 2, stream));
    }
  } else {
    for (float** p : {&f->p_hi, &f->p_lo}) {
      if (XKNN_PCONV && p == &f->p_lo) continue;
      XK_CUDA(dalloc(p, pb));
      XK_CUDA(cudaMemsetAsync(*p, 0, pb * 4, stream));
    }
  }
  XK_CUDA(dalloc(&f->partial_f, (uint64_t)2 * (f->mwpad / 256) * f->bpad));
  XK_CUDA(dalloc(&f->labelterm, f->bpad));
  f->dx_units_cap = 148ull * 256;
  XK_CUDA(dalloc(&f->partial_dx, f->dx_units_cap * 512));
  XK_CUDA(dalloc(&f->dW32, wb));
  XK_CUDA(dalloc(&f->dw_part, (uint64_t)kNumSMs / 2 * 256 * 512));
  XK_CUDA(dalloc(&f->lab_head, f->mwpad));
  XK_CUDA(cudaMemsetAsync(f->lab_head, 0xff, (uint64_t)f->mwpad * 4, stream));
  XK_CUDA(dalloc(&f->lab_next, f->bpad));
  XK_CUDA(dalloc(&dXpart, (uint64_t)f->bpad * d));
  const auto S128 = CU_TENSOR_MAP_SWIZZLE_128B, S64 = CU_TENSOR_MAP_SWIZZLE_64B;
  const auto S32G = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;  // MN-major tf32 operands
  bool ok = true;
  constexpr uint32_t FKB = Cfg3<kF3>::KB;
  const auto SF = FKB == 32 ? S128 : S64;
  if (f->mixed) {  // tf32 rows and the bf16 planes, KB x 128 boxes
    constexpr uint32_t MKB = Cfg3<kFm>::KB;
    const auto ST = MKB == 32 ? S128 : S64, SB = MKB == 32 ? S64 : CU_TENSOR_MAP_SWIZZLE_32B;
    ok &= make_map32(&f->mF_Ah, f->xh_hi, 512, f->bpad, MKB, 128, ST);
    ok &= make_map32(&f->mF_Al, f->xb_hi, 512, f->bpad, MKB, 128, SB, true);
    ok &= make_map32(&f->mF_Ad, f->xd, 512, f->bpad, MKB, 128, SB, true);
    ok &= make_map32(&f->mF_Bh, f->w_hi, 512, f->mwpad, MKB, 128, ST);
    ok &= make_map32(&f->mF_Bl, f->wb_hi, 512, f->mwpad, MKB, 128, SB, true);
    ok &= make_map32(&f->mF_Bd, f->wd, 512, f->mwpad, MKB, 128, SB, true);
  } else {
    ok &= make_map32(&f->mF_Ah, f->xh_hi, 512, f->bpad, FKB, 128, SF);
    ok &= make_map32(&f->mF_Al, f->xh_lo, 512, f->bpad, FKB, 128, SF);
    ok &= make_map32(&f->mF_Bh, f->w_hi, 512, f->mwpad, FKB, 128, SF);
    ok &= make_map32(&f->mF_Bl, f->w_lo, 512, f->mwpad, FKB, 128, SF);
    f->mF_Ad = f->mF_Ah;
    f->mF_Bd = f->mF_Bh;
  }
  if (f->bfb) {  // bf16 planes in the BF16 path's layouts (fast.cu), 32 K per stage
    ok &= make_map32(&f->mDX_Ah, f->pb_hi, f->mwpad, f->bpad, 32, 128, S64, true);
    ok &= make_map32(&f->mDX_Al, f->pb_lo, f->mwpad, f->bpad, 32, 128, S64, true);
    ok &= make_map32(&f->mDX_Bh, f->wb_hi, 512, f->mwpad, 64, 32, S128, true);
    ok &= make_map32(&f->mDX_Bl, f->wb_lo, 512, f->mwpad, 64, 32, S128, true);
    ok &= make_map32(&f->mDW_Ah, f->pb_hi, f->mwpad, f->bpad, 64, 32, S128, true);
    ok &= make_map32(&f->mDW_Al, f->pb_lo, f->mwpad, f->bpad, 64, 32, S128, true);
    ok &= make_map32(&f->mDW_Bh, f->xsb_hi, 512, f->bpad, 64, 32, S128, true);
    ok &= make_map32(&f->mDW_Bl, f->xsb_lo, 512, f->bpad, 64, 32, S128, true);
  } else {
    ok &= make_map32(&f->mDX_Ah, f->p_hi, f->mwpad, f->bpad, 16, 128, S64);
    float* plo = XKNN_PCONV ? f->p_hi : f->p_lo;  // (unused when the consumers split P~)
    ok &= make_map32(&f->mDX_Al, plo, f->mwpad, f->bpad, 16, 128, S64);
    ok &= make_map32(&f->mDX_Bh, f->w_hi, 512, f->mwpad, 32, 16, S32G);
    ok &= make_map32(&f->mDX_Bl, f->w_lo, 512, f->mwpad, 32, 16, S32G);
    ok &= make_map32(&f->mDW_Ah, f->p_hi, f->mwpad, f->bpad, 32, 16, S32G);
    ok &= make_map32(&f->mDW_Al, plo, f->mwpad, f->bpad, 32, 16, S32G);
    ok &= make_map32(&f->mDW_Bh, f->xs_hi, 512, f->bpad, 32, 16, S32G);
    ok &= make_map32(&f->mDW_Bl, f->xs_lo, 512, f->bpad, 32, 16, S32G);
  }
  ok &= make_map32(&f->mDX_st, f->partial_dx, 512, f->dx_units_cap, 32, 32, S128);
  ok &= make_map32(&f->mDW_st, f->dW32, 512, f->mwpad, 32, 32, S128);
  ok &= make_map32(&f->mDWP_st, f->dw_part, 512, (uint64_t)kNumSMs / 2 * 256, 32, 32, S128);
  if (!ok) return fail_msg(XKNN_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  XK_CUDA(cudaFuncSetAttribute(k_gemm3<kF3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes3<kF3>()));
  XK_CUDA(cudaFuncSetAttribute(k_gemm3<kDX3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes3<kDX3>()));
  XK_CUDA(cudaFuncSetAttribute(k_gemm3<kDW3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes3<kDW3>()));
  XK_CUDA(cudaFuncSetAttribute(k_gemm3<kFm>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes3<kFm>()));
  XK_CUDA(cudaFuncSetAttribute(k_gemm3<kDXb>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes3<kDXb>()));
  XK_CUDA(cudaFuncSetAttribute(k_gemm3<kDWb>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes3<kDWb>()));
  XK_CUDA(cudaFuncSetAttribute(k_gemm3<kDWh>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem_bytes3<kDWh>()));
  return XKNN_OK;
}

void Layer::free_fast32() {
  auto* f = static_cast<Fast32State*>(fast32);
  if (!f) return;
  for (void* p : {(void*)f->xh_hi, (void*)f->xh_lo, (void*)f->xs_hi, (void*)f->xs_lo,
                  (void*)f->w_hi, (void*)f->w_lo, (void*)f->p_hi, (void*)f->p_lo,
                  (void*)f->partial_f, (void*)f->labelterm, (void*)f->partial_dx, (void*)f->dW32,
                  (void*)f->dw_part, (void*)f->lab_head, (void*)f->lab_next, (void*)f->pb_hi,
                  (void*)f->pb_lo, (void*)f->wb_hi, (void*)f->wb_lo, (void*)f->xsb_hi,
                  (void*)f->xsb_lo, (void*)f->xb_hi, (void*)f->xd, (void*)f->wd})
    if (p) cudaFree(p);
  delete f;
  fast32 = nullptr;
}

xknn_status_t Layer::reset_fast32_scratch() {
  auto* f = static_cast<Fast32State*>(fast32);
  if (!f) return XKNN_OK;
  XK_CUDA(cudaMemsetAsync(f->lab_head, 0xff, (uint64_t)f->mwpad * 4, stream));
  return XKNN_OK;
}

xknn_status_t Layer::run_fast32_core(uint64_t B) {
  auto* f = static_cast<Fast32State*>(fast32);
  const uint32_t D = (uint32_t)d;
  if (B > f->bpad) return XKNN_ERR_INVALID_ARGUMENT;
  // (a) operands: the active weight rows gathered + normalized, split hi/lo (feature all-gather
  //     runs under it at P > 1), then X_hat hi/lo
  XK_CUDA(launch_normalize_rows(W, mw_cap, D, active, &st->active_count, begin, f->w_hi, f->wb_hi,
                                wnorm, err, stream, false, f->w_lo, f->wb_lo, f->wd));
  ++launches;
  launch_pdl(k_zero_rows32, 64, 256, 0, stream, (const SelState*)st, f->w_hi, f->w_lo, f->wb_hi,
             f->wb_lo, f->mwpad);
  XK_LAUNCH();
  if (world > 1) XK_TRY(wait_features());
  XK_CUDA(launch_normalize_rows(X, B, D, nullptr, nullptr, 0, f->xh_hi, f->xb_hi, xnorm, err,
                                stream, false, f->mixed ? nullptr : f->xh_lo, nullptr, f->xd));
  ++launches;
  mark(3);
  Gemm3Args ga{};
  ga.st = st;
  ga.B = (uint32_t)B;
  ga.bpad = f->bpad;
  ga.scale = cfg.scale;
  ga.label_col = label_col;
  ga.p_hi = f->p_hi;
  ga.p_lo = f->p_lo;
  ga.pb_hi = f->pb_hi;
  ga.pb_lo = f->pb_lo;
  ga.ldp = ldp;
  ga.labelterm = f->labelterm;
  const uint32_t nbp = (uint32_t)((B + 255) / 256);
  // (b) GEMM-F with the fused exp / row-sum / label-logit epilogue
  ga.partial = f->partial_f;
  ga.nbt = nbp;
  ga.splits = gemm_pair_splits(nbp, 1u << 30);
  if (f->mixed)
    launch_pdl_cluster(k_gemm3<kFm>, kNumSMs, 384, smem_bytes3<kFm>(), stream, 2u, f->mF_Ah,
                       f->mF_Al, f->mF_Bh, f->mF_Bl, f->mF_Ah, f->mF_Ah, f->mF_Ad, f->mF_Bd, ga);
  else
    launch_pdl_cluster(k_gemm3<kF3>, kNumSMs, 384, smem_bytes3<kF3>(), stream, 2u, f->mF_Ah,
                       f->mF_Al, f->mF_Bh, f->mF_Bl, f->mF_Ah, f->mF_Ah, f->mF_Ah, f->mF_Ah, ga);
  XK_LAUNCH();
  mark(4);
  // (c) row statistics -> all-reduce over the class shards -> (d) loss, X_hat', label lists
  XK_CUDA(launch_rowreduce(st, f->partial_f, f->labelterm, label_col, (uint32_t)B, f->bpad, rowred,
                           stream));
  ++launches;
  if (world > 1) {
    if (par_ar.ready) {
      XK_CUDA(par_ar.launch(rowred, 3 * B, err, stream));
      ++launches;
    } else {
      XK_NCCL(ncclAllReduce(rowred, rowred, 3 * B, ncclDouble, ncclSum, comm, stream));
    }
  }
  launch_pdl(k_fixup32, grid_for((uint64_t)f->bpad * 32, 256), 256, 0, stream, (const double*)rowred,
             (const int32_t*)label_col, (const float*)X, (const float*)xnorm, (uint32_t)B, f->bpad,
             cfg.scale, f->lab_head, f->lab_next, f->xs_hi, f->xs_lo, f->xsb_hi, f->xsb_lo, loss_dev,
             st, err);
  XK_LAUNCH();
  mark(5);
  // (e) GEMM-dW -> fp32 dW rows (compact active order)
  if (f->bfb && XKNN_DWH)
    launch_pdl_cluster(k_gemm3<kDWh>, kNumSMs, 384, smem_bytes3<kDWh>(), stream, 2u, f->mDW_Ah,
                       f->mDW_Al, f->mDW_Bh, f->mDW_Bl, f->mDW_st, f->mDWP_st, f->mDW_st,
                       f->mDW_st, ga);
  else if (f->bfb)
    launch_pdl_cluster(k_gemm3<kDWb>, kNumSMs, 384, smem_bytes3<kDWb>(), stream, 2u, f->mDW_Ah,
                       f->mDW_Al, f->mDW_Bh, f->mDW_Bl, f->mDW_st, f->mDWP_st, f->mDW_st,
                       f->mDW_st, ga);
  else
    launch_pdl_cluster(k_gemm3<kDW3>, kNumSMs, 384, smem_bytes3<kDW3>(), stream, 2u, f->mDW_Ah,
                       f->mDW_Al, f->mDW_Bh, f->mDW_Bl, f->mDW_st, f->mDWP_st, f->mDW_st,
                       f->mDW_st, ga);
  XK_LAUNCH();
  mark(6);
  // (f) GEMM-dX split-K partials -> reduce (+ one-hot correction) -> reduce-scatter
  ga.partial = f->partial_dx;
  const uint32_t dx_splits = gemm_pair_splits(nbp, 148);
  ga.nbt = nbp;
  ga.splits = dx_splits;
  if (f->bfb)
    launch_pdl_cluster(k_gemm3<kDXb>, kNumSMs, 384, smem_bytes3<kDXb>(), stream, 2u, f->mDX_Ah,
                       f->mDX_Al, f->mDX_Bh, f->mDX_Bl, f->mDX_st, f->mDX_st, f->mDX_st,
                       f->mDX_st, ga);
  else
    launch_pdl_cluster(k_gemm3<kDX3>, kNumSMs, 384, smem_bytes3<kDX3>(), stream, 2u, f->mDX_Ah,
                       f->mDX_Al, f->mDX_Bh, f->mDX_Bl, f->mDX_st, f->mDX_st, f->mDX_st,
                       f->mDX_st, ga);
  XK_LAUNCH();
  mark(7);
  XK_CUDA(launch_dx_reduce(f->partial_dx, rowred, (uint32_t)B, nbp, dx_splits, cfg.scale,
                           label_col, active, begin, W, wnorm, world > 1 ? dXpart : dX, stream));
  ++launches;
  const uint64_t bl = B / world;
  if (world > 1) {
    XK_CUDA(cudaEventRecord(ev_fork, stream));
    XK_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
    XK_NCCL(ncclReduceScatter(dXpart, dX, bl * d, ncclFloat, ncclSum, comm, side));
    XK_CUDA(cudaEventRecord(ev_join, side));
  }
  // (g) normalize-backward + momentum SGD on the active rows, with the one-hot correction
  mark(8);
  // (tail-unit K-partials: every dW kind but the half-width one)
  LabelFix lf{f->lab_head, f->lab_next, X, xnorm, (float)((double)cfg.scale / (double)B),
              f->bfb && XKNN_DWH ? nullptr : f->dw_part, (uint32_t)kNumSMs / 2};
  XK_CUDA(launch_update_rows(W, V, f->dW32, active, &st->active_count, mw_cap, begin, D, wnorm,
                             lr_dev, cfg.momentum, cfg.weight_decay, err, stream, 148u * 16u, lf));
  ++launches;
  if (world > 1) XK_CUDA(cudaStreamWaitEvent(stream, ev_join, 0));
  return XKNN_OK;
}

}  // namespace xknn
static_assert(xknn::smem_bytes3<xknn::kF3>() <= 232448, "GEMM-F tf32 pair smem");
static_assert(xknn::smem_bytes3<xknn::kDX3>() <= 232448, "GEMM-dX tf32 pair smem");
static_assert(xknn::smem_bytes3<xknn::kDW3>() <= 232448, "GEMM-dW tf32 pair smem");
static_assert(xknn::smem_bytes3<xknn::kDXb>() <= 232448, "GEMM-dX bf16x3 pair smem");
static_assert(xknn::smem_bytes3<xknn::kFm>() <= 232448, "GEMM-F mixed pair smem");
static_assert(xknn::smem_bytes3<xknn::kDWb>() <= 232448, "GEMM-dW bf16x3 pair smem");
static_assert(xknn::smem_bytes3<xknn::kDWh>() <= 232448, "GEMM-dW bf16x3 half-unit pair smem");
