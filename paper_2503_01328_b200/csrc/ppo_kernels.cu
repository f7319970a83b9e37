// libppo_b200.so -- recompute kernels K3 (LayerNorm), K4 (GeLU), K5 (Philox dropout).
//
// These are the "trivial layers" whose recompute shrinks the saved set from 34bsh to
// 20bsh per layer (reference pkg/src/ppoff/costs.py:1-7,18-20).  All are
// HBM-bound: one CTA row-loop per LayerNorm row with one 16-byte bf16x8 vector per
// thread, grid-stride 16-byte vectors for the elementwise ops.
#include "ppo_common.cuh"

namespace ppo {

constexpr int kMaxHidden = 8192;  // hidden/8 threads per row, <= 1024

__device__ __forceinline__ void load_params8(const float* p, int t, float (&out)[8]) {
  const float4* v = reinterpret_cast<const float4*>(p + 8 * t);
  float4 a = v[0], b = v[1];
  out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
  out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
}

// out = resid + dropout(branch) (or out := x when resid == nullptr);  ln = LN(out).
template <bool kResidual>
__global__ void __launch_bounds__(1024) ln_fwd_kernel(const __nv_bfloat16* __restrict__ resid,
                                                      const __nv_bfloat16* __restrict__ src,
                                                      __nv_bfloat16* __restrict__ out,
                                                      const float* __restrict__ gamma,
                                                      const float* __restrict__ beta,
                                                      __nv_bfloat16* __restrict__ ln, int64_t rows,
                                                      int hidden, float eps, uint32_t threshold,
                                                      float scale, uint64_t seed, uint64_t offset,
                                                      int use_dropout) {
  __shared__ float scratch[32 * 2];
  const int t = threadIdx.x;
  const bool active = t < (hidden >> 3);
  float gm[8], bt[8];
  if (active && ln) {
    load_params8(gamma, t, gm);
    load_params8(beta, t, bt);
  }
  const float inv_h = 1.f / (float)hidden;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t base = row * hidden + 8 * t;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0.f;
    if (active) {
      if (kResidual) {
        float r[8], b[8];
        unpack8(ld_stream(resid + base), r);
        unpack8(ld_stream(src + base), b);
        uint32_t keep = use_dropout ? keep_mask8((uint64_t)base, seed, offset, threshold) : 0xFFu;
        const float sc = use_dropout ? scale : 1.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = bf16_round(r[i] + (((keep >> i) & 1u) ? b[i] * sc : 0.f));
        st_stream(out + base, pack8(v));
      } else {
        unpack8(ld_stream(src + base), v);
      }
    }
    if (!ln) continue;
    float s1[1] = {0.f};
#pragma unroll
    for (int i = 0; i < 8; ++i) s1[0] += v[i];
    block_sum<1>(s1, scratch);
    const float mean = s1[0] * inv_h;
    float s2[1] = {0.f};
    if (active) {
#pragma unroll
      for (int i = 0; i < 8; ++i) s2[0] += (v[i] - mean) * (v[i] - mean);
    }
    block_sum<1>(s2, scratch);
    const float rstd = rsqrtf(s2[0] * inv_h + eps);
    if (active) {
      float y[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) y[i] = (v[i] - mean) * rstd * gm[i] + bt[i];
      st_stream(ln + base, pack8(y));
    }
  }
}

// dx = resid_grad + LN_bwd(dy; x) with mean/rstd recomputed from x;
// dgamma/dbeta accumulated per CTA then one atomic per column;
// drop_out = dropout_bwd(bf16(dx)) when requested.
__global__ void __launch_bounds__(1024) ln_bwd_kernel(
    const __nv_bfloat16* __restrict__ x, const float* __restrict__ gamma,
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ resid_grad,
    __nv_bfloat16* __restrict__ dx, float* __restrict__ dgamma, float* __restrict__ dbeta,
    int64_t rows, int hidden, float eps, __nv_bfloat16* __restrict__ drop_out, uint32_t threshold,
    float scale, uint64_t seed, uint64_t offset) {
  __shared__ float scratch[32 * 3];
  const int t = threadIdx.x;
  const bool active = t < (hidden >> 3);
  float gm[8], acc_g[8], acc_b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc_g[i] = acc_b[i] = gm[i] = 0.f;
  if (active) load_params8(gamma, t, gm);
  const float inv_h = 1.f / (float)hidden;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t base = row * hidden + 8 * t;
    float xv[8], g[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) xv[i] = g[i] = 0.f;
    if (active) {
      unpack8(ld_stream(x + base), xv);
      unpack8(ld_stream(dy + base), g);
    }
    float s1[1] = {0.f};
#pragma unroll
    for (int i = 0; i < 8; ++i) s1[0] += xv[i];
    block_sum<1>(s1, scratch);
    const float mean = s1[0] * inv_h;
    float s3[3] = {0.f, 0.f, 0.f};
    float dyv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      dyv[i] = g[i];
      const float c = active ? xv[i] - mean : 0.f;
      xv[i] = c;  // centred
      g[i] = g[i] * gm[i];
      s3[0] += c * c;
      s3[1] += g[i];
      s3[2] += g[i] * c;
    }
    block_sum<3>(s3, scratch);
    const float rstd = rsqrtf(s3[0] * inv_h + eps);
    const float mg = s3[1] * inv_h;                 // mean(g)
    const float mgx = s3[2] * rstd * inv_h;         // mean(g * xhat)
    if (active) {
      float d[8], rg[8];
      if (resid_grad) unpack8(ld_stream(resid_grad + base), rg);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xhat = xv[i] * rstd;
        d[i] = bf16_round(rstd * (g[i] - mg - xhat * mgx) + (resid_grad ? rg[i] : 0.f));
        acc_g[i] += dyv[i] * xhat;
        acc_b[i] += dyv[i];
      }
      st_stream(dx + base, pack8(d));
      if (drop_out) {
        const uint32_t keep = keep_mask8((uint64_t)base, seed, offset, threshold);
#pragma unroll
        for (int i = 0; i < 8; ++i) d[i] = ((keep >> i) & 1u) ? d[i] * scale : 0.f;
        st_stream(drop_out + base, pack8(d));
      }
    }
  }
  if (active) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      atomicAdd(dgamma + 8 * t + i, acc_g[i]);
      atomicAdd(dbeta + 8 * t + i, acc_b[i]);
    }
  }
}

__global__ void dropout_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                               int64_t n8, uint32_t threshold, float scale, uint64_t seed,
                               uint64_t offset) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n8;
       c += (int64_t)gridDim.x * blockDim.x) {
    float v[8];
    unpack8(ld_stream(x + 8 * c), v);
    const uint32_t keep = keep_mask8((uint64_t)(8 * c), seed, offset, threshold);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = ((keep >> i) & 1u) ? v[i] * scale : 0.f;
    st_stream(y + 8 * c, pack8(v));
  }
}

// gelu_tanh(x) = 0.5 x (1 + tanh(k0 (x + k1 x^3)))
__device__ __forceinline__ void gelu_and_grad(float x, float& g, float& dg) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float x2 = x * x;
  const float u = k0 * x * fmaf(k1, x2, 1.f);
  const float th = tanhf(u);
  g = 0.5f * x * (1.f + th);
  dg = 0.5f * (1.f + th) + 0.5f * x * (1.f - th * th) * k0 * fmaf(3.f * k1, x2, 1.f);
}

__global__ void gelu_fwd_kernel(const __nv_bfloat16* __restrict__ f, __nv_bfloat16* __restrict__ g,
                                int64_t n8) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n8;
       c += (int64_t)gridDim.x * blockDim.x) {
    float v[8];
    unpack8(ld_stream(f + 8 * c), v);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float gg, dd;
      gelu_and_grad(v[i], gg, dd);
      v[i] = gg;
    }
    st_stream(g + 8 * c, pack8(v));
  }
}

__global__ void gelu_bwd_kernel(const __nv_bfloat16* __restrict__ f, const __nv_bfloat16* dg_in,
                                __nv_bfloat16* __restrict__ g_out, __nv_bfloat16* df_out, int64_t n8) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n8;
       c += (int64_t)gridDim.x * blockDim.x) {
    float v[8], d[8], gg[8];
    unpack8(ld_stream(f + 8 * c), v);
    unpack8(*reinterpret_cast<const uint4*>(dg_in + 8 * c), d);
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

__global__ void colsum_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ acc, int64_t rows,
                              int64_t cols, int64_t rows_per_block) {
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

static int check_rows(const char* who, int64_t rows, int64_t hidden) {
  if (rows < 0 || hidden <= 0 || (hidden & 7) || hidden > kMaxHidden)
    return set_error(PPO_ESHAPE, "%s: hidden=%lld must be a positive multiple of 8 <= %d", who,
                     (long long)hidden, kMaxHidden);
  return PPO_OK;
}

static int row_threads(int64_t hidden) { return (int)(((hidden >> 3) + 31) / 32 * 32); }

static int elementwise_grid(int64_t n8) {
  const int64_t cap = (int64_t)sm_count_current() * 8;
  int64_t want = (n8 + 255) / 256;
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace ppo

using namespace ppo;

extern "C" {

int ppo_layernorm_fwd(const void* x, const float* gamma, const float* beta, void* y, int64_t rows,
                      int64_t hidden, float eps, void* stream) {
  if (int rc = check_rows("ppo_layernorm_fwd", rows, hidden)) return rc;
  if (!x || !gamma || !beta || !y) return set_error(PPO_EINVAL, "ppo_layernorm_fwd: null pointer");
  if (rows == 0) return PPO_OK;
  const int grid = (int)(rows < (int64_t)sm_count_current() * 16 ? rows : (int64_t)sm_count_current() * 16);
  ln_fwd_kernel<false><<<grid, row_threads(hidden), 0, as_stream(stream)>>>(
      nullptr, static_cast<const __nv_bfloat16*>(x), nullptr, gamma, beta, static_cast<__nv_bfloat16*>(y), rows,
      (int)hidden, eps, 0u, 1.f, 0, 0, 0);
  PPO_LAUNCHED("ln_fwd_kernel");
  return PPO_OK;
}

int ppo_residual_dropout_ln_fwd(const void* resid, const void* branch, void* out, const float* gamma,
                                const float* beta, void* ln, int64_t rows, int64_t hidden, float eps,
                                float p, uint64_t seed, uint64_t offset, void* stream) {
  if (int rc = check_rows("ppo_residual_dropout_ln_fwd", rows, hidden)) return rc;
  if (!resid || !branch || !out || (ln && (!gamma || !beta)))
    return set_error(PPO_EINVAL, "ppo_residual_dropout_ln_fwd: null pointer");
  if (!(p >= 0.f && p < 1.f)) return set_error(PPO_EINVAL, "ppo_residual_dropout_ln_fwd: p=%f", p);
  if (rows == 0) return PPO_OK;
  const int grid = (int)(rows < (int64_t)sm_count_current() * 16 ? rows : (int64_t)sm_count_current() * 16);
  ln_fwd_kernel<true><<<grid, row_threads(hidden), 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(resid), static_cast<const __nv_bfloat16*>(branch),
      static_cast<__nv_bfloat16*>(out), gamma, beta, static_cast<__nv_bfloat16*>(ln), rows, (int)hidden, eps,
      dropout_threshold(p), 1.f / (1.f - p), seed, offset, p > 0.f ? 1 : 0);
  PPO_LAUNCHED("ln_fwd_kernel<residual>");
  return PPO_OK;
}

int ppo_layernorm_bwd(const void* x, const float* gamma, const void* dy, const void* resid_grad, void* dx,
                      float* dgamma, float* dbeta, int64_t rows, int64_t hidden, float eps, void* drop_out,
                      float p, uint64_t drop_seed, uint64_t drop_offset, void* stream) {
  if (int rc = check_rows("ppo_layernorm_bwd", rows, hidden)) return rc;
  if (!x || !gamma || !dy || !dx || !dgamma || !dbeta)
    return set_error(PPO_EINVAL, "ppo_layernorm_bwd: null pointer");
  if (!(p >= 0.f && p < 1.f)) return set_error(PPO_EINVAL, "ppo_layernorm_bwd: p=%f", p);
  if (rows == 0) return PPO_OK;
  // Few CTAs with a row loop: the dgamma/dbeta atomics scale with the grid.
  const int64_t cap = (int64_t)sm_count_current() * (hidden <= 2048 ? 4 : 2);
  const int grid = (int)(rows < cap ? rows : cap);
  ln_bwd_kernel<<<grid, row_threads(hidden), 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), gamma, static_cast<const __nv_bfloat16*>(dy),
      static_cast<const __nv_bfloat16*>(resid_grad), static_cast<__nv_bfloat16*>(dx), dgamma, dbeta, rows,
      (int)hidden, eps, static_cast<__nv_bfloat16*>(drop_out), dropout_threshold(p), p > 0.f ? 1.f / (1.f - p) : 1.f,
      drop_seed, drop_offset);
  PPO_LAUNCHED("ln_bwd_kernel");
  return PPO_OK;
}

int ppo_dropout(const void* x, void* y, int64_t n, float p, uint64_t seed, uint64_t offset, void* stream) {
  if (!x || !y || n < 0 || (n & 7)) return set_error(PPO_EINVAL, "ppo_dropout: bad arguments (n %% 8 != 0?)");
  if (!(p >= 0.f && p < 1.f)) return set_error(PPO_EINVAL, "ppo_dropout: p=%f", p);
  if (n == 0) return PPO_OK;
  const int64_t n8 = n >> 3;
  dropout_kernel<<<elementwise_grid(n8), 256, 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), n8, dropout_threshold(p),
      1.f / (1.f - p), seed, offset);
  PPO_LAUNCHED("dropout_kernel");
  return PPO_OK;
}

int ppo_gelu_fwd(const void* f, void* g, int64_t n, void* stream) {
  if (!f || !g || n < 0 || (n & 7)) return set_error(PPO_EINVAL, "ppo_gelu_fwd: bad arguments");
  if (n == 0) return PPO_OK;
  gelu_fwd_kernel<<<elementwise_grid(n >> 3), 256, 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(f), static_cast<__nv_bfloat16*>(g), n >> 3);
  PPO_LAUNCHED("gelu_fwd_kernel");
  return PPO_OK;
}

int ppo_gelu_bwd(const void* f, const void* dg, void* g, void* df, int64_t n, void* stream) {
  if (!f || !dg || !df || n < 0 || (n & 7)) return set_error(PPO_EINVAL, "ppo_gelu_bwd: bad arguments");
  if (n == 0) return PPO_OK;
  gelu_bwd_kernel<<<elementwise_grid(n >> 3), 256, 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(f), static_cast<const __nv_bfloat16*>(dg), static_cast<__nv_bfloat16*>(g),
      static_cast<__nv_bfloat16*>(df), n >> 3);
  PPO_LAUNCHED("gelu_bwd_kernel");
  return PPO_OK;
}

int ppo_colsum(const void* x, float* acc, int64_t rows, int64_t cols, void* stream) {
  if (!x || !acc || rows < 0 || cols <= 0 || (cols & 7)) return set_error(PPO_EINVAL, "ppo_colsum: bad arguments");
  if (rows == 0) return PPO_OK;
  const int threads = 128;
  const int64_t gx = (cols / 8 + threads - 1) / threads;
  const int64_t rpb = 64;
  const int64_t gy = (rows + rpb - 1) / rpb;
  colsum_kernel<<<dim3((unsigned)gx, (unsigned)gy), threads, 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), acc, rows, cols, rpb);
  PPO_LAUNCHED("colsum_kernel");
  return PPO_OK;
}

}  // extern "C"
