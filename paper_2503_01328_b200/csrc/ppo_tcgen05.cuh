// Shared tcgen05 / TMA / mbarrier building blocks of the hand-written attention kernels
// (K7 forward, K7b backward).  Internal header of libppo_b200.so.
#pragma once

#include <cuda.h>  // CUtensorMap; the encoder comes from cudaGetDriverEntryPoint

#include <mutex>

#include "ppo_common.cuh"

namespace ppo {
namespace tc {

constexpr int kHalf = 128 * 64 * 2;  // one 128-row x 64-column bf16 TMA box (16 KB)

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// one lane of a converged warp (the UMMA warp runs converged so its operands stay uniform)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, 0xffffffff;\n@px mov.s32 %0, 1;\n}\n"
      : "+r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  if (elect_one())
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns; thread t gets lane (base lane + t).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (x <= 0): round-to-nearest split through the 1.5 * 2^23 shifter,
// degree-3 fit of 2^f on [-1/2, 1/2] (max relative error 1.4e-4, far below the bf16
// rounding P gets for the tensor core), exponent added as an integer.  A share of the
// softmax exponentials runs here so the SFU (16 results per clock per SM) stops being
// the bound of the P phase.
__device__ __forceinline__ float ex2_fma(float x) {
  x = fmaxf(x, -126.f);
  const float j = x + 12582912.f;
  const float f = x - (j - 12582912.f);
  const float q = fmaf(fmaf(fmaf(0.0550292665f, f, 0.242256982f), f, 0.693253055f), f, 0.999951339f);
  return __int_as_float(__float_as_int(q) + (__float_as_int(j) << 23));
}

// ---- packed fp32 pairs (Blackwell FFMA2 / FADD2) and 3-input max
__device__ __forceinline__ uint64_t f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f2u(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// ex2_fma on a pair with the arithmetic in packed FFMA2 / FADD2 (x <= 0).
__device__ __forceinline__ float2 ex2_fma2(float x0, float x1) {
  const uint64_t x = f2(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const uint64_t j = fadd2(x, f2(12582912.f, 12582912.f));
  const uint64_t t = fadd2(j, f2(-12582912.f, -12582912.f));
  const uint64_t f = ffma2(t, f2(-1.f, -1.f), x);
  uint64_t q = ffma2(f2(0.0550292665f, 0.0550292665f), f, f2(0.242256982f, 0.242256982f));
  q = ffma2(q, f, f2(0.693253055f, 0.693253055f));
  q = ffma2(q, f, f2(0.999951339f, 0.999951339f));
  const float2 qq = f2u(q), jj = f2u(j);
  return make_float2(__int_as_float(__float_as_int(qq.x) + (__float_as_int(jj.x) << 23)),
                     __int_as_float(__float_as_int(qq.y) + (__float_as_int(jj.y) << 23)));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return reinterpret_cast<uint32_t&>(v);
}

// UMMA shared-memory descriptors for a 128 x 128 bf16 tile stored as two 64-column halves
// (16 KB apart), 128 B per row, 128-byte swizzle (the TMA SWIZZLE_128B box layout).
//   K-major (rows = M/N, columns = K):  SBO = 1024 B between 8-row groups; the k-th
//     16-element step starts 32 B further inside the swizzle atom (next half at k = 4).
//   MN-major (rows = K, columns = M/N): LBO = 16 KB between the 64-wide M/N halves,
//     SBO = 1024 B between 8-row K groups; the k-th 16-row step starts 2 KB further.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// instruction descriptor: bf16 x bf16 -> f32, M = 128
__host__ __device__ constexpr uint32_t idesc(uint32_t a_mn, uint32_t b_mn, uint32_t n = 128) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

// One 128 x N x (16 kSteps) GEMM = kSteps UMMAs of K = 16, issued by one elected lane of the
// converged UMMA warp.  a4 / b4: shared-memory tile start >> 4 (descriptor address field),
// or for kATmem the TMEM address of A (K = 16 per 8 columns of bf16 pairs).  Descriptor low
// words are a4/b4 + compile-time constants (no carry: addresses < 2^18); the high word is
// SBO = 1024 B, version 1, SWIZZLE_128B for both majors.
template <int kSteps, bool kAMn, bool kBMn, bool kATmem, int kBHalf = kHalf>
__device__ __forceinline__ void gemm128(uint32_t d, uint32_t a4, uint32_t b4, uint32_t idesc, bool acc) {
  asm volatile("" : "+r"(a4), "+r"(b4));  // keep the per-k descriptors out of the loop-invariant pool
  constexpr uint64_t kHi = uint64_t(0x40004040u) << 32;
  if (elect_one()) {
#pragma unroll
    for (int k = 0; k < kSteps; ++k) {
      const uint32_t boff = kBMn ? (k * 2048) >> 4 : (((k >> 2) * kBHalf + (k & 3) * 32) >> 4);
      const uint64_t bd = kHi | (b4 + boff + (kBMn ? (uint32_t(kBHalf) >> 4) << 16 : 1u << 16));
      const uint32_t en = (acc || k > 0) ? 1u : 0u;
      if constexpr (kATmem) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
            "r"(a4 + k * 8), "l"(bd), "r"(idesc), "r"(en)
            : "memory");
      } else {
        const uint32_t aoff = kAMn ? (k * 2048) >> 4 : (((k >> 2) * kHalf + (k & 3) * 32) >> 4);
        const uint64_t ad = kHi | (a4 + aoff + (kAMn ? (uint32_t(kHalf) >> 4) << 16 : 1u << 16));
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(en)
            : "memory");
      }
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------------ host side
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiled encoder(int* rc) {
  static std::once_flag once;
  static EncodeTiled fn = nullptr;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(f);
  });
  *rc = fn ? PPO_OK : set_error(PPO_ENOTSUP, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 3-D map over a row-major [rows][heads][D] view: dims (D, heads, rows), 128-byte swizzle.
inline int make_map(EncodeTiled enc, CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base, int D,
                    uint64_t heads, uint64_t rows, uint64_t row_stride_bytes, uint32_t box_d, uint32_t box_rows) {
  cuuint64_t dims[3] = {uint64_t(D), heads, rows};
  cuuint64_t strides[2] = {uint64_t(D) * esize, row_stride_bytes};
  cuuint32_t box[3] = {box_d, 1, box_rows};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(PPO_EINVAL, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return PPO_OK;
}

}  // namespace tc
}  // namespace ppo
