// libppo_b200.so -- recompute kernels K4 (GeLU), K5 (Philox dropout) and column sums.
// LayerNorm (K3) lives in ppo_layernorm.cu.
//
// These are the "trivial layers" whose recompute shrinks the saved set from 34bsh to
// 20bsh per layer (reference pkg/src/ppoff/costs.py:1-7,18-20).  All are
// HBM-bound elementwise ops: grid-stride loops over 16-byte bf16x8 vectors.
#include "ppo_common.cuh"

namespace ppo {

__global__ void __launch_bounds__(256) dropout_kernel(const __nv_bfloat16* __restrict__ x,
                                                      __nv_bfloat16* __restrict__ y, int64_t n8,
                                                      uint32_t threshold, float scale, uint64_t seed,
                                                      uint64_t offset_add, const uint64_t* __restrict__ offset_base) {
  pdl_wait();
  const uint64_t offset = offset_add + (offset_base ? __ldg(offset_base) : 0ull);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c0 < n8; c0 += 2 * stride) {
    uint4 raw[2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (c0 + u * stride < n8) raw[u] = ld_stream(x + 8 * (c0 + u * stride));
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t c = c0 + u * stride;
      if (c >= n8) break;
      float v[8];
      unpack8(raw[u], v);
      const uint32_t keep = keep_mask8((uint64_t)(8 * c), seed, offset, threshold);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = ((keep >> i) & 1u) ? v[i] * scale : 0.f;
      st_stream(y + 8 * c, pack8(v));
    }
  }
}

// Elementwise kernels move two bf16x8 vectors per thread per iteration (grid stride),
// all loads of an iteration issued before any math.
constexpr int kVec = 2;

__global__ void __launch_bounds__(256) gelu_fwd_kernel(const __nv_bfloat16* __restrict__ f,
                                                       __nv_bfloat16* __restrict__ g, int64_t n8) {
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c0 < n8; c0 += kVec * stride) {
    uint4 raw[kVec];
#pragma unroll
    for (int u = 0; u < kVec; ++u)
      if (c0 + u * stride < n8) raw[u] = ld_stream(f + 8 * (c0 + u * stride));
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      const int64_t c = c0 + u * stride;
      if (c >= n8) break;
      float v[8];
      unpack8(raw[u], v);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float gg, dd;
        gelu_and_grad(v[i], gg, dd);
        v[i] = gg;
      }
      st_stream(g + 8 * c, pack8(v));
    }
  }
}

__global__ void __launch_bounds__(256) gelu_bwd_kernel(const __nv_bfloat16* __restrict__ f,
                                                       const __nv_bfloat16* dg_in,
                                                       __nv_bfloat16* __restrict__ g_out,
                                                       __nv_bfloat16* df_out, int64_t n8) {
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c0 < n8; c0 += kVec * stride) {
    uint4 rf[kVec], rd[kVec];
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      const int64_t c = c0 + u * stride;
      if (c < n8) {
        rf[u] = ld_stream(f + 8 * c);
        rd[u] = *reinterpret_cast<const uint4*>(dg_in + 8 * c);  // may alias df_out
      }
    }
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      const int64_t c = c0 + u * stride;
      if (c >= n8) break;
      float v[8], d[8], gg[8];
      unpack8(rf[u], v);
      unpack8(rd[u], d);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float dd;
        gelu_and_grad(v[i], gg[i], dd);
        d[i] *= dd;
      }
      if (g_out) st_stream(g_out + 8 * c, pack8(gg));
      *reinterpret_cast<uint4*>(df_out + 8 * c) = pack8(d);
    }
  }
}

__global__ void colsum_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ acc, int64_t rows,
                              int64_t cols, int64_t rows_per_block) {
  pdl_wait();
  const int64_t col8 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (8 * col8 >= cols) return;
  const int64_t r0 = blockIdx.y * rows_per_block;
  const int64_t r1 = r0 + rows_per_block < rows ? r0 + rows_per_block : rows;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int64_t r = r0; r < r1; ++r) {
    float v[8];
    unpack8(ld_stream(x + r * cols + 8 * col8), v);
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i] += v[i];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) atomicAdd(acc + 8 * col8 + i, s[i]);
}

// Token + position embedding of the first stage: x[r] = wte[tok[r]] + wpe[r]
// (bf16 sum rounded once, as torch's embedding + add).  One warp per row, 16-B
// vectors; the token ids are read from device memory so the launch can sit in a
// CUDA graph whose token row changes between replays.
__global__ void __launch_bounds__(256) embed_fwd_kernel(const int64_t* __restrict__ tok,
                                                        const __nv_bfloat16* __restrict__ wte,
                                                        const __nv_bfloat16* __restrict__ wpe,
                                                        __nv_bfloat16* __restrict__ x, int64_t rows, int64_t h,
                                                        int64_t vocab) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t n8 = h >> 3;
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    int64_t t = __ldg(tok + r);
    t = t < 0 ? 0 : (t >= vocab ? vocab - 1 : t);
    const __nv_bfloat16* a = wte + t * h;
    const __nv_bfloat16* b = wpe + r * h;
    for (int64_t c = lane; c < n8; c += 32) {
      float va[8], vb[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(a) + c), va);
      unpack8(ld_stream(b + 8 * c), vb);
#pragma unroll
      for (int i = 0; i < 8; ++i) va[i] += vb[i];
      st_stream(x + r * h + 8 * c, pack8(va));
    }
  }
}

// Embedding backward: gwte[tok[r]] += dy[r] and gwpe[r] += dy[r] in fp32, straight
// from the bf16 gradient (no fp32 copy of dy); 16-byte vector atomics
// (red.global.add.v4.f32) -- repeated tokens in a row add in arbitrary order, as
// torch's index_add_.
__global__ void __launch_bounds__(256) embed_bwd_kernel(const int64_t* __restrict__ tok,
                                                        const __nv_bfloat16* __restrict__ dy,
                                                        float* __restrict__ gwte, float* __restrict__ gwpe,
                                                        int64_t rows, int64_t h, int64_t vocab) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t n8 = h >> 3;
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    int64_t t = __ldg(tok + r);
    t = t < 0 ? 0 : (t >= vocab ? vocab - 1 : t);
    for (int64_t c = lane; c < n8; c += 32) {
      float v[8];
      unpack8(ld_stream(dy + r * h + 8 * c), v);
      float4* e = reinterpret_cast<float4*>(gwte + t * h + 8 * c);
      float4* p = reinterpret_cast<float4*>(gwpe + r * h + 8 * c);
      atomicAdd(e, make_float4(v[0], v[1], v[2], v[3]));
      atomicAdd(e + 1, make_float4(v[4], v[5], v[6], v[7]));
      atomicAdd(p, make_float4(v[0], v[1], v[2], v[3]));
      atomicAdd(p + 1, make_float4(v[4], v[5], v[6], v[7]));
    }
  }
}

static int row_grid(int64_t rows) {
  const int64_t cap = (int64_t)sm_count_current() * 8;  // 8 CTAs of 8 warps per SM
  const int64_t want = (rows + 7) / 8;
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

static int elementwise_grid(int64_t n8) {
  const int64_t cap = (int64_t)sm_count_current() * 8;
  int64_t want = (n8 + 511) / 512;
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

template <typename K>
static int set_smem(K kernel, size_t bytes) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return cuda_error(e, "cudaFuncSetAttribute(smem)");
  return PPO_OK;
}

}  // namespace ppo

using namespace ppo;

extern "C" {

int ppo_dropout(const void* x, void* y, int64_t n, float p, uint64_t seed, uint64_t offset,
                const uint64_t* offset_base, void* stream) {
  if (!x || !y || n < 0 || (n & 7)) return set_error(PPO_EINVAL, "ppo_dropout: bad arguments (n %% 8 != 0?)");
  if (!(p >= 0.f && p < 1.f)) return set_error(PPO_EINVAL, "ppo_dropout: p=%f", p);
  if (n == 0) return PPO_OK;
  const int64_t n8 = n >> 3;
  launch_pdl(dropout_kernel, elementwise_grid(n8), 256, 0, as_stream(stream), 
      static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), n8, dropout_threshold(p),
      1.f / (1.f - p), seed, offset, offset_base);
  PPO_LAUNCHED("dropout_kernel");
  return PPO_OK;
}

int ppo_gelu_fwd(const void* f, void* g, int64_t n, void* stream) {
  if (!f || !g || n < 0 || (n & 7)) return set_error(PPO_EINVAL, "ppo_gelu_fwd: bad arguments");
  if (n == 0) return PPO_OK;
  launch_pdl(gelu_fwd_kernel, elementwise_grid(n >> 3), 256, 0, as_stream(stream),
      static_cast<const __nv_bfloat16*>(f), static_cast<__nv_bfloat16*>(g), n >> 3);
  PPO_LAUNCHED("gelu_fwd_kernel");
  return PPO_OK;
}

int ppo_gelu_bwd(const void* f, const void* dg, void* g, void* df, int64_t n, void* stream) {
  if (!f || !dg || !df || n < 0 || (n & 7)) return set_error(PPO_EINVAL, "ppo_gelu_bwd: bad arguments");
  if (n == 0) return PPO_OK;
  launch_pdl(gelu_bwd_kernel, elementwise_grid(n >> 3), 256, 0, as_stream(stream),
      static_cast<const __nv_bfloat16*>(f), static_cast<const __nv_bfloat16*>(dg), static_cast<__nv_bfloat16*>(g),
      static_cast<__nv_bfloat16*>(df), n >> 3);
  PPO_LAUNCHED("gelu_bwd_kernel");
  return PPO_OK;
}

int ppo_embed_fwd(const int64_t* tokens, const void* wte, const void* wpe, void* x, int64_t rows, int64_t hidden,
                  int64_t vocab, void* stream) {
  if (!tokens || !wte || !wpe || !x || rows < 0 || hidden <= 0 || (hidden & 7) || vocab <= 0)
    return set_error(PPO_EINVAL, "ppo_embed_fwd: bad arguments (hidden %% 8 != 0?)");
  if (!aligned16(wte) || !aligned16(wpe) || !aligned16(x)) return set_error(PPO_EINVAL, "ppo_embed_fwd: unaligned");
  if (rows == 0) return PPO_OK;
  launch_pdl(embed_fwd_kernel, row_grid(rows), 256, 0, as_stream(stream), 
      tokens, static_cast<const __nv_bfloat16*>(wte), static_cast<const __nv_bfloat16*>(wpe),
      static_cast<__nv_bfloat16*>(x), rows, hidden, vocab);
  PPO_LAUNCHED("embed_fwd_kernel");
  return PPO_OK;
}

int ppo_embed_bwd(const int64_t* tokens, const void* dy, float* gwte, float* gwpe, int64_t rows, int64_t hidden,
                  int64_t vocab, void* stream) {
  if (!tokens || !dy || !gwte || !gwpe || rows < 0 || hidden <= 0 || (hidden & 7) || vocab <= 0)
    return set_error(PPO_EINVAL, "ppo_embed_bwd: bad arguments (hidden %% 8 != 0?)");
  if (!aligned16(dy) || !aligned16(gwte) || !aligned16(gwpe)) return set_error(PPO_EINVAL, "ppo_embed_bwd: unaligned");
  if (rows == 0) return PPO_OK;
  launch_pdl(embed_bwd_kernel, row_grid(rows), 256, 0, as_stream(stream), 
      tokens, static_cast<const __nv_bfloat16*>(dy), gwte, gwpe, rows, hidden, vocab);
  PPO_LAUNCHED("embed_bwd_kernel");
  return PPO_OK;
}

int ppo_colsum(const void* x, float* acc, int64_t rows, int64_t cols, void* stream) {
  if (!x || !acc || rows < 0 || cols <= 0 || (cols & 7)) return set_error(PPO_EINVAL, "ppo_colsum: bad arguments");
  if (rows == 0) return PPO_OK;
  const int threads = 128;
  const int64_t gx = (cols / 8 + threads - 1) / threads;
  const int64_t rpb = 64;
  const int64_t gy = (rows + rpb - 1) / rpb;
  launch_pdl(colsum_kernel, dim3((unsigned)gx, (unsigned)gy), threads, 0, as_stream(stream), 
      static_cast<const __nv_bfloat16*>(x), acc, rows, cols, rpb);
  PPO_LAUNCHED("colsum_kernel");
  return PPO_OK;
}

}  // extern "C"
