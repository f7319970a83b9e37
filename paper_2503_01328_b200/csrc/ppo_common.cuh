// Shared helpers of libppo_b200.so: error plumbing, launch accounting, bf16 vectors,
// Philox4x32-10.  Internal header; the ABI is include/ppo_b200.h.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <utility>
#include <cstdarg>
#include <cstdio>

#include "../../include/ppo_b200.h"

namespace ppo {

int set_error(int code, const char* fmt, ...);
int cuda_error(cudaError_t err, const char* what);
int sm_count_current();
extern std::atomic<uint64_t> g_launches;

inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

#define PPO_TRY_CUDA(expr)                                  \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return ::ppo::cuda_error(_e, #expr); \
  } while (0)

// Checks the launch that was just enqueued (configuration errors only).
#define PPO_LAUNCHED(name)                                  \
  do {                                                      \
    ::ppo::count_launch();                                  \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return ::ppo::cuda_error(_e, name); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------ programmatic dependent launch
// Every kernel of the library starts with pdl_wait() (griddepcontrol.wait: returns once
// the preceding kernel on the stream has completed and its memory is visible; a no-op
// for a normal launch) and is launched through launch_pdl, which sets the PDL attribute
// when PPO_PDL has bit 0 set (bit 1: the CUTLASS GEMMs, whose GDC waits are compiled
// in).  Default off: measured 1.5-3.5% slower per iteration at C2 in every mode,
// whole-iteration CUDA graph (profiles/r1_pdl_ab.jsonl).
int pdl_mode();  // PPO_PDL bit 0: our kernels, bit 1: CUTLASS GEMMs
inline bool pdl_enabled() { return (pdl_mode() & 1) != 0; }
inline bool pdl_gemm_enabled() { return (pdl_mode() & 2) != 0; }

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
inline cudaEvent_t as_event(void* e) { return reinterpret_cast<cudaEvent_t>(e); }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ------------------------------------------------------------------ bf16 x 8
struct alignas(16) Bf16x8 {
  __nv_bfloat162 h[4];
};

__device__ __forceinline__ void unpack8(const uint4& raw, float (&f)[8]) {
  const Bf16x8& v = reinterpret_cast<const Bf16x8&>(raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(v.h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  Bf16x8 v;
#pragma unroll
  for (int i = 0; i < 4; ++i) v.h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return reinterpret_cast<const uint4&>(v);
}

// Round-trip through bf16 so math sees exactly what was stored.
__device__ __forceinline__ float bf16_round(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w));
}

// gelu_tanh(x) = 0.5 x (1 + tanh(k0 (x + k1 x^3))); tanh on the SFU (tanh.approx.f32,
// ~2^-11 relative error, far below the bf16 output rounding of 2^-8).
__device__ __forceinline__ float fast_tanh(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void gelu_and_grad(float x, float& g, float& dg) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float x2 = x * x;
  const float u = k0 * x * fmaf(k1, x2, 1.f);
  const float th = fast_tanh(u);
  g = 0.5f * x * (1.f + th);
  dg = 0.5f * (1.f + th) + 0.5f * x * (1.f - th * th) * k0 * fmaf(3.f * k1, x2, 1.f);
}

// ------------------------------------------------------------ Philox4x32-10
struct U32x4 {
  uint32_t v[4];
};

__host__ __device__ __forceinline__ void mulhilo(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umulhi(a, b);
#else
  uint64_t p = (uint64_t)a * (uint64_t)b;
  lo = (uint32_t)p;
  hi = (uint32_t)(p >> 32);
#endif
}

// counter (c0..c3), key (k0, k1); ten rounds, Random123 constants.
__host__ __device__ __forceinline__ U32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                        uint32_t c3, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo(M0, c0, hi0, lo0);
    mulhilo(M1, c2, hi1, lo1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += W0;
    k1 += W1;
  }
  U32x4 out;
  out.v[0] = c0;
  out.v[1] = c1;
  out.v[2] = c2;
  out.v[3] = c3;
  return out;
}

// Keep bits for elements e0 .. e0+7 (e0 % 8 == 0) of tensor (seed, offset): one
// Philox4x32-10 block per 8 elements, one 16-bit lane per element (low half of word
// i/2 for even i, high half for odd i); kept iff lane >= threshold16 = floor(p * 2^16).
__device__ __forceinline__ uint32_t keep_mask8(uint64_t e0, uint64_t seed, uint64_t offset,
                                               uint32_t threshold16) {
  const uint64_t ctr = e0 >> 3;
  const U32x4 r = philox4x32_10((uint32_t)ctr, (uint32_t)(ctr >> 32), (uint32_t)offset,
                                (uint32_t)(offset >> 32), (uint32_t)seed, (uint32_t)(seed >> 32));
  uint32_t bits = 0;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    bits |= ((r.v[w] & 0xFFFFu) >= threshold16 ? 1u : 0u) << (2 * w);
    bits |= ((r.v[w] >> 16) >= threshold16 ? 1u : 0u) << (2 * w + 1);
  }
  return bits;
}

// floor(p * 2^16), clamped; p in [0, 1).
inline uint32_t dropout_threshold(float p) {
  double t = (double)p * 65536.0;
  if (t <= 0.0) return 0u;
  if (t >= 65535.0) return 65535u;
  return (uint32_t)t;
}

// ------------------------------------------------------------ block reductions
// Sums N values across the block; every thread gets the totals.  `scratch` holds
// 33*N floats.  Two barriers: warp partials -> per-value reduction by N threads ->
// broadcast.  Safe to call back to back (the caller's next write to scratch is
// after the final barrier of this call).
template <int N>
__device__ __forceinline__ void block_sum(float (&v)[N], float* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  if (nwarps == 1) return;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) scratch[warp * N + i] = v[i];
  }
  __syncthreads();
  if (threadIdx.x < N) {
    float t = 0.f;
    for (int w = 0; w < nwarps; ++w) t += scratch[w * N + threadIdx.x];
    scratch[32 * N + threadIdx.x] = t;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = scratch[32 * N + i];
  __syncthreads();
}

// ------------------------------------------------------ TMA bulk copies + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Order earlier generic-proxy shared-memory accesses before later async-proxy (TMA) writes.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 1-D TMA: global -> shared, completion counted on `bar` (bytes % 16 == 0, 16 B aligned).
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 1-D TMA: shared -> global, tracked by the issuing thread's bulk async-group.
__device__ __forceinline__ void tma_store_1d(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// Wait until at most N committed store groups still read shared memory.
template <int N>
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

// Wait until every committed store group has completed (writes visible).
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace ppo
