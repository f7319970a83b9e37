// libppo_b200.so -- K3: LayerNorm forward / backward with residual-add and Philox dropout
// fused in, the recomputed "trivial layer" of the 34bsh -> 20bsh saved set
// (reference pkg/src/ppoff/costs.py:1-7,18-20).
//
// Warp-group-per-row design.  A row of h bf16 is owned by W = ceil(h / (256 VPL))
// warps; lane L of the group holds vectors v = L + 32W*j (j < VPL) of 8 bf16 each, so
// every warp access is a fully coalesced 512-byte sweep and a lane keeps VPL x (number
// of input tensors) independent 16-byte loads in flight.  Row statistics need only warp
// shuffles (plus one named barrier when W > 1) -- no block-wide barrier inside the
// row loop.  Statistics are one-pass (sum, sum of squares) in fp32.  The LayerNorm
// parameter gradients accumulate in registers (a lane owns fixed columns), are folded
// per CTA in shared memory and flushed with 16-byte vector atomics.
#include "ppo_common.cuh"

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>

namespace ppo {

constexpr int kMaxHidden = 8192;
constexpr int kGroupsPerBlock = 4;  // rows processed concurrently by one CTA (at most)

// Rows per CTA for a W-warp row group: up to 4, but never more than 16 warps per CTA, so
// 32*W*G threads leave >= 128 registers a thread (fewer spill the double-buffered rows).
constexpr int groups_for(int W) { return (16 / W) > kGroupsPerBlock ? kGroupsPerBlock : ((16 / W) < 1 ? 1 : 16 / W); }
// The forward kernels hold fewer live registers: 4 rows per CTA up to 5-warp rows (measured
// 9% faster than 3 at h = 5120), the register-safe count above that.
constexpr int fwd_groups_for(int W) { return W <= 5 ? kGroupsPerBlock : groups_for(W); }

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Sum N values over the W warps of a row group; every lane gets the totals.
template <int W, int N>
__device__ __forceinline__ void group_sum(float (&v)[N], float* scratch, int group) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  if constexpr (W > 1) {
    const int wig = (threadIdx.x >> 5) % W;  // warp index inside the group
    float* s = scratch + group * W * N;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
      for (int i = 0; i < N; ++i) s[wig * N + i] = v[i];
    }
    named_sync(1 + group, 32 * W);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < W; ++w) t += s[w * N + i];
      v[i] = t;
    }
    named_sync(1 + group, 32 * W);
  }
}

// 8 consecutive fp32 parameters through the read-only path (L1-resident after the
// first row: every CTA reads the same h floats).
__device__ __forceinline__ void load8f(const float* p, float (&o)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}

// out = resid + dropout(branch)  (kResidual)  or  v = src  (!kResidual);  ln = LN(v).
// The next row's vectors are requested before the current row is reduced, so DRAM
// latency overlaps the shuffle reduction and the stores (register double-buffering).
//
// kDual (no residual): two independent LayerNorms in one launch -- rows [0, rows_a) are
// LN(src) * gamma + beta -> ln, rows [rows_a, rows) are LN(resid) * gamma_b + beta_b -> out
// (the W pass's LN1 and LN2 recompute: one 4E launch instead of two 2E launches).
template <bool kResidual, int W, int kVecPerLane, int G, bool kDual = false, int kMinBlocks = 1>
__global__ void __launch_bounds__(32 * W * G, kMinBlocks > 1 ? kMinBlocks : 0) ln_fwd_kernel(
    const __nv_bfloat16* __restrict__ resid, const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ out,
    const float* __restrict__ gamma, const float* __restrict__ beta, __nv_bfloat16* __restrict__ ln, int64_t rows,
    int hidden, float eps, uint32_t threshold, float scale, uint64_t seed, uint64_t offset_add,
    const uint64_t* __restrict__ offset_base, int use_dropout, const float* __restrict__ gamma_b,
    const float* __restrict__ beta_b, int64_t rows_a) {
  static_assert(!(kDual && kResidual), "dual LayerNorm has no residual");
  pdl_wait();
  extern __shared__ __align__(16) float sm[];
  const uint64_t offset = offset_add + (offset_base ? __ldg(offset_base) : 0ull);
  float* scratch = sm;
  const int group = threadIdx.x / (32 * W);
  const int L = threadIdx.x % (32 * W);
  const int nvec = hidden >> 3;
  const float inv_h = 1.f / (float)hidden;
  const int64_t step = (int64_t)gridDim.x * G;
  int64_t row = (int64_t)blockIdx.x * G + group;
  uint4 ra[kVecPerLane], rb[kVecPerLane];
  auto fetch = [&](int64_t r, uint4 (&a)[kVecPerLane], uint4 (&b)[kVecPerLane]) {
#pragma unroll
    for (int j = 0; j < kVecPerLane; ++j) {
      const int v = L + 32 * W * j;
      if (v < nvec) {
        if (kDual)
          b[j] = ld_stream(r < rows_a ? src + r * hidden + 8 * v : resid + (r - rows_a) * hidden + 8 * v);
        else
          b[j] = ld_stream(src + r * hidden + 8 * v);
        if (kResidual) a[j] = ld_stream(resid + r * hidden + 8 * v);
      }
    }
  };
  if (row < rows) fetch(row, ra, rb);
  for (; row < rows; row += step) {
    const int64_t rbase = row * hidden;
    uint4 na[kVecPerLane], nb[kVecPerLane];
    if (row + step < rows) fetch(row + step, na, nb);
    float sums[2] = {0.f, 0.f};
#pragma unroll
    for (int j = 0; j < kVecPerLane; ++j) {
      const int v = L + 32 * W * j;
      if (v >= nvec) continue;
      float val[8];
      if (kResidual) {
        float a[8], b[8];
        unpack8(ra[j], a);
        unpack8(rb[j], b);
        const uint32_t keep = use_dropout ? keep_mask8((uint64_t)(rbase + 8 * v), seed, offset, threshold) : 0xFFu;
        const float sc = use_dropout ? scale : 1.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) val[i] = a[i] + (((keep >> i) & 1u) ? b[i] * sc : 0.f);
        rb[j] = pack8(val);  // keep the stored bf16 bits; LN reads exactly what was stored
        st_stream(out + rbase + 8 * v, rb[j]);
      }
      unpack8(rb[j], val);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        sums[0] += val[i];
        sums[1] += val[i] * val[i];
      }
    }
    if (ln) {
      group_sum<W, 2>(sums, scratch, group);
      const float mean = sums[0] * inv_h;
      const float rstd = rsqrtf(fmaxf(sums[1] * inv_h - mean * mean, 0.f) + eps);
      const bool second = kDual && row >= rows_a;
      const float* gm = second ? gamma_b : gamma;
      const float* bt = second ? beta_b : beta;
      __nv_bfloat16* dst = second ? out + (rbase - rows_a * hidden) : ln + rbase;
#pragma unroll
      for (int j = 0; j < kVecPerLane; ++j) {
        const int v = L + 32 * W * j;
        if (v >= nvec) continue;
        float val[8], g[8], b[8], y[8];
        unpack8(rb[j], val);
        load8f(gm + 8 * v, g);
        load8f(bt + 8 * v, b);
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = (val[i] - mean) * rstd * g[i] + b[i];
        st_stream(dst + 8 * v, pack8(y));
      }
    }
#pragma unroll
    for (int j = 0; j < kVecPerLane; ++j) {
      ra[j] = na[j];
      rb[j] = nb[j];
    }
  }
}

// dx = resid_grad + LN_bwd(dy; x) (statistics recomputed from x);
// dgamma += sum_rows dy*xhat, dbeta += sum_rows dy;  drop_out = dropout_bwd(bf16(dx));
// kLnOut: ln_out = LN(x) * gamma + beta -- the LayerNorm RECOMPUTE the weight gradient of
// the GEMM that consumed LN(x) in the forward needs, emitted from the statistics and the
// x already in registers: one extra write instead of a separate read-x / write-ln
// kernel (K3 fused into the backward).
//
// A lane owns the same kVecPerLane x 8 columns on every row it visits, so the
// parameter-gradient sums live in registers for the whole row loop; at the end the
// CTA's row groups are folded in shared memory and flushed with one 16-byte vector
// atomic per 4 columns.  kPrefetch: the next row's vectors are requested before the
// current row is reduced (register double-buffering).  (Shared-memory accumulation per
// row and shared-memory staging of gamma were measured 1.6-3x slower / spilling,
// profiles/r2_ln_bwd_variants.jsonl.)
template <int W, int kVecPerLane, int G, bool kLnOut, bool kPrefetch>
__global__ void __launch_bounds__(32 * W * G) ln_bwd_kernel(
    const __nv_bfloat16* __restrict__ x, const float* __restrict__ gamma, const float* __restrict__ beta,
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ resid_grad, __nv_bfloat16* __restrict__ dx,
    float* __restrict__ dgamma, float* __restrict__ dbeta, __nv_bfloat16* __restrict__ ln_out, int64_t rows,
    int hidden, float eps, __nv_bfloat16* __restrict__ drop_out, uint32_t threshold, float scale, uint64_t seed,
    uint64_t offset_add, const uint64_t* __restrict__ offset_base) {
  pdl_wait();
  extern __shared__ __align__(16) float sm[];
  const uint64_t offset = offset_add + (offset_base ? __ldg(offset_base) : 0ull);
  float* s_acc = sm;                 // [2h]: dgamma partials, then dbeta partials
  float* scratch = sm + 2 * hidden;  // group reductions
  const int group = threadIdx.x / (32 * W);
  const int L = threadIdx.x % (32 * W);
  const int nvec = hidden >> 3;
  const float inv_h = 1.f / (float)hidden;
  const bool has_resid = resid_grad != nullptr;
  const int64_t step = (int64_t)gridDim.x * G;
  float acc_g[kVecPerLane][8], acc_b[kVecPerLane][8];
#pragma unroll
  for (int j = 0; j < kVecPerLane; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc_g[j][i] = acc_b[j][i] = 0.f;
  uint4 rx[kVecPerLane], rd[kVecPerLane], rr[kVecPerLane];
  auto fetch = [&](int64_t r, uint4 (&a)[kVecPerLane], uint4 (&b)[kVecPerLane], uint4 (&c)[kVecPerLane]) {
#pragma unroll
    for (int j = 0; j < kVecPerLane; ++j) {
      const int v = L + 32 * W * j;
      if (v < nvec) {
        a[j] = ld_stream(x + r * hidden + 8 * v);
        b[j] = ld_stream(dy + r * hidden + 8 * v);
        if (has_resid) c[j] = ld_stream(resid_grad + r * hidden + 8 * v);
      }
    }
  };
  int64_t row = (int64_t)blockIdx.x * G + group;
  if (kPrefetch && row < rows) fetch(row, rx, rd, rr);
  for (; row < rows; row += step) {
    const int64_t rbase = row * hidden;
    uint4 nx[kPrefetch ? kVecPerLane : 1], nd[kPrefetch ? kVecPerLane : 1], nr[kPrefetch ? kVecPerLane : 1];
    if constexpr (kPrefetch) {
      if (row + step < rows) fetch(row + step, nx, nd, nr);
    } else {
      fetch(row, rx, rd, rr);
    }
    float sums[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < kVecPerLane; ++j) {
      const int v = L + 32 * W * j;
      if (v >= nvec) continue;
      float xv[8], dv[8], g[8];
      unpack8(rx[j], xv);
      unpack8(rd[j], dv);
      load8f(gamma + 8 * v, g);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float gi = dv[i] * g[i];
        sums[0] += xv[i];
        sums[1] += xv[i] * xv[i];
        sums[2] += gi;
        sums[3] += gi * xv[i];
      }
    }
    group_sum<W, 4>(sums, scratch, group);
    const float mean = sums[0] * inv_h;
    const float rstd = rsqrtf(fmaxf(sums[1] * inv_h - mean * mean, 0.f) + eps);
    const float mg = sums[2] * inv_h;                        // mean(g)
    const float mgx = rstd * (sums[3] * inv_h - mean * mg);  // mean(g * xhat)
#pragma unroll
    for (int j = 0; j < kVecPerLane; ++j) {
      const int v = L + 32 * W * j;
      if (v >= nvec) continue;
      float xv[8], dv[8], g[8], rg[8], d[8];
      unpack8(rx[j], xv);
      unpack8(rd[j], dv);
      load8f(gamma + 8 * v, g);
      if (has_resid) unpack8(rr[j], rg);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = (xv[i] - mean) * rstd;
        d[i] = rstd * (dv[i] * g[i] - mg - xh * mgx) + (has_resid ? rg[i] : 0.f);
        acc_g[j][i] += dv[i] * xh;
        acc_b[j][i] += dv[i];
      }
      if constexpr (kLnOut) {
        float b[8];
        load8f(beta + 8 * v, b);
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[i] = (xv[i] - mean) * rstd * g[i] + b[i];
        st_stream(ln_out + rbase + 8 * v, pack8(xv));
      }
      const uint4 packed = pack8(d);
      st_stream(dx + rbase + 8 * v, packed);
      if (drop_out) {
        unpack8(packed, d);  // the replay applies to the stored bf16 gradient
        const uint32_t keep = keep_mask8((uint64_t)(rbase + 8 * v), seed, offset, threshold);
#pragma unroll
        for (int i = 0; i < 8; ++i) d[i] = ((keep >> i) & 1u) ? d[i] * scale : 0.f;
        st_stream(drop_out + rbase + 8 * v, pack8(d));
      }
    }
    if constexpr (kPrefetch) {
#pragma unroll
      for (int j = 0; j < kVecPerLane; ++j) {
        rx[j] = nx[j];
        rd[j] = nd[j];
        rr[j] = nr[j];
      }
    }
  }
  // fold the row groups of this CTA in shared memory, one group at a time
  for (int gi = 0; gi < G; ++gi) {
    if (group == gi) {
#pragma unroll
      for (int j = 0; j < kVecPerLane; ++j) {
        const int v = L + 32 * W * j;
        if (v >= nvec) continue;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float pg = gi ? s_acc[8 * v + i] : 0.f;
          const float pb = gi ? s_acc[hidden + 8 * v + i] : 0.f;
          s_acc[8 * v + i] = pg + acc_g[j][i];
          s_acc[hidden + 8 * v + i] = pb + acc_b[j][i];
        }
      }
    }
    __syncthreads();
  }
  for (int c = 4 * threadIdx.x; c < hidden; c += 4 * blockDim.x) {
    atomicAdd(reinterpret_cast<float4*>(dgamma + c), *reinterpret_cast<const float4*>(s_acc + c));
    atomicAdd(reinterpret_cast<float4*>(dbeta + c), *reinterpret_cast<const float4*>(s_acc + hidden + c));
  }
}

static int check_rows(const char* who, int64_t rows, int64_t hidden) {
  if (rows < 0 || hidden <= 0 || (hidden & 7) || hidden > kMaxHidden)
    return set_error(PPO_ESHAPE, "%s: hidden=%lld must be a positive multiple of 8 <= %d", who,
                     (long long)hidden, kMaxHidden);
  return PPO_OK;
}

// Vectors per lane per tensor.  Fewer vectors per lane means more warps per row:
// these kernels are latency-bound at transformer sizes (one row is a short dependent
// chain), so parallelism across warps beats per-lane ILP.  PPO_LN_VPL overrides (2/4/8)
// for A/B runs.
static int vpl_choice(int64_t hidden, int dflt) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("PPO_LN_VPL");
    env = e ? atoi(e) : 0;
  }
  int v = (env == 2 || env == 4 || env == 8) ? env : dflt;
  while (v < 8 && (hidden + 256 * v - 1) / (256 * v) > 8) v *= 2;  // at most 8 warps per row
  return v;
}

// PPO_LN_FWD_MINB=4: forward LayerNorm kernels compiled for >= 4 resident CTAs per SM
// (register cap 64 at 256 threads) -- an occupancy A/B for the latency-bound C2 shapes.
static bool ln_fwd_min4() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PPO_LN_FWD_MINB");
    v = (e && atoi(e) == 4) ? 1 : 0;
  }
  return v == 1;
}

static int warps_per_row(int64_t hidden, int vpl) { return (int)((hidden + 256 * vpl - 1) / (256 * vpl)); }

struct RowLaunch {
  int grid, block;
  size_t smem;
};

// Grid = every row group resident at once when the occupancy allows, else one full
// wave of resident CTAs (148 SMs x CTAs per SM) looping over the rows.
template <typename K>
static int row_launch(K kernel, int64_t rows, int64_t hidden, int W, int param_arrays, RowLaunch* l,
                      int groups_per_block = kGroupsPerBlock) {
  l->block = 32 * W * groups_per_block;
  l->smem = (size_t)param_arrays * hidden * sizeof(float) + (size_t)groups_per_block * W * 4 * sizeof(float);
  // The occupancy query and smem attribute are host work on every launch otherwise;
  // cache them per (device, kernel, block, smem).
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, reinterpret_cast<const void*>(kernel), l->block, l->smem);
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) per_sm = it->second;
  }
  if (per_sm == 0) {
    if (l->smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)l->smem);
      if (e != cudaSuccess) return cuda_error(e, "cudaFuncSetAttribute(smem)");
    }
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, l->block, l->smem);
    if (e != cudaSuccess) return cuda_error(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    if (per_sm < 1) per_sm = 1;
    std::lock_guard<std::mutex> lock(mu);
    cache[key] = per_sm;
  }
  const int64_t groups = (rows + groups_per_block - 1) / groups_per_block;
  const int64_t cap = (int64_t)sm_count_current() * (per_sm > 0 ? per_sm : 1);
  l->grid = (int)(groups < cap ? (groups > 0 ? groups : 1) : cap);
  return PPO_OK;
}


}  // namespace ppo

using namespace ppo;

extern "C" {

#define PPO_VPL_DISPATCH(VPL_, MACRO) \
  switch (VPL_) {                     \
    case 2: MACRO(2) break;           \
    case 4: MACRO(4) break;           \
    default: MACRO(8) break;          \
  }

int ppo_layernorm_fwd(const void* x, const float* gamma, const float* beta, void* y, int64_t rows, int64_t hidden,
                      float eps, void* stream) {
  if (int rc = check_rows("ppo_layernorm_fwd", rows, hidden)) return rc;
  if (!x || !gamma || !beta || !y) return set_error(PPO_EINVAL, "ppo_layernorm_fwd: null pointer");
  if (rows == 0) return PPO_OK;
  RowLaunch l;
  int rc = PPO_OK;
  const int vpl = vpl_choice(hidden, 4);
#define PPO_LN_FWD_K(W, V, MB)                                                                                \
  if ((rc = row_launch(ln_fwd_kernel<false, W, V, fwd_groups_for(W), false, MB>, rows, hidden, W, 0, &l,      \
                       fwd_groups_for(W)))) return rc;                                                         \
  launch_pdl(ln_fwd_kernel<false, W, V, fwd_groups_for(W), false, MB>, l.grid, l.block, l.smem,                \
      as_stream(stream), nullptr, static_cast<const __nv_bfloat16*>(x), nullptr, gamma, beta,                  \
      static_cast<__nv_bfloat16*>(y), rows, (int)hidden, eps, 0u, 1.f, 0, 0, nullptr, 0, nullptr, nullptr,      \
      (int64_t)0);
#define PPO_LN_FWD_W(W, V)                                \
  if (ln_fwd_min4()) { PPO_LN_FWD_K(W, V, 4) } else { PPO_LN_FWD_K(W, V, 1) }
#define PPO_LN_FWD_V(V)                                               \
  {                                                                   \
    switch (warps_per_row(hidden, V)) {                               \
      case 1: PPO_LN_FWD_W(1, V) break;                               \
      case 2: PPO_LN_FWD_W(2, V) break;                               \
      case 3: PPO_LN_FWD_W(3, V) break;                               \
      case 4: PPO_LN_FWD_W(4, V) break;                               \
      case 5: PPO_LN_FWD_W(5, V) break;                               \
      case 6: PPO_LN_FWD_W(6, V) break;                               \
      case 7: PPO_LN_FWD_W(7, V) break;                               \
      default: PPO_LN_FWD_W(8, V) break;                              \
    }                                                                 \
  }
  PPO_VPL_DISPATCH(vpl, PPO_LN_FWD_V)
#undef PPO_LN_FWD_V
#undef PPO_LN_FWD_W
#undef PPO_LN_FWD_K
  PPO_LAUNCHED("ln_fwd_kernel");
  return PPO_OK;
}

int ppo_residual_dropout_ln_fwd(const void* resid, const void* branch, void* out, const float* gamma,
                                const float* beta, void* ln, int64_t rows, int64_t hidden, float eps, float p,
                                uint64_t seed, uint64_t offset, const uint64_t* offset_base, void* stream) {
  if (int rc = check_rows("ppo_residual_dropout_ln_fwd", rows, hidden)) return rc;
  if (!resid || !branch || !out || (ln && (!gamma || !beta)))
    return set_error(PPO_EINVAL, "ppo_residual_dropout_ln_fwd: null pointer");
  if (!(p >= 0.f && p < 1.f)) return set_error(PPO_EINVAL, "ppo_residual_dropout_ln_fwd: p=%f", p);
  if (rows == 0) return PPO_OK;
  RowLaunch l;
  int rc = PPO_OK;
  const int vpl = vpl_choice(hidden, 4);
#define PPO_RES_K(W, V, MB)                                                                                   \
  if ((rc = row_launch(ln_fwd_kernel<true, W, V, fwd_groups_for(W), false, MB>, rows, hidden, W, 0, &l,       \
                       fwd_groups_for(W)))) return rc;                                                         \
  launch_pdl(ln_fwd_kernel<true, W, V, fwd_groups_for(W), false, MB>, l.grid, l.block, l.smem,                 \
      as_stream(stream), static_cast<const __nv_bfloat16*>(resid), static_cast<const __nv_bfloat16*>(branch),  \
      static_cast<__nv_bfloat16*>(out), gamma, beta, static_cast<__nv_bfloat16*>(ln), rows, (int)hidden, eps,   \
      dropout_threshold(p), 1.f / (1.f - p), seed, offset, offset_base, p > 0.f ? 1 : 0, nullptr, nullptr,      \
      (int64_t)0);
#define PPO_RES_W(W, V)                                   \
  if (ln_fwd_min4()) { PPO_RES_K(W, V, 4) } else { PPO_RES_K(W, V, 1) }
#define PPO_RES_V(V)                                                  \
  {                                                                   \
    switch (warps_per_row(hidden, V)) {                               \
      case 1: PPO_RES_W(1, V) break;                                  \
      case 2: PPO_RES_W(2, V) break;                                  \
      case 3: PPO_RES_W(3, V) break;                                  \
      case 4: PPO_RES_W(4, V) break;                                  \
      case 5: PPO_RES_W(5, V) break;                                  \
      case 6: PPO_RES_W(6, V) break;                                  \
      case 7: PPO_RES_W(7, V) break;                                  \
      default: PPO_RES_W(8, V) break;                                 \
    }                                                                 \
  }
  PPO_VPL_DISPATCH(vpl, PPO_RES_V)
#undef PPO_RES_V
#undef PPO_RES_W
#undef PPO_RES_K
  PPO_LAUNCHED("ln_fwd_kernel<residual>");
  return PPO_OK;
}

// PPO_LN_BWD=1: no next-row prefetch (A/B runs; tools/ln_bwd_sweep.py)
static bool ln_bwd_prefetch() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PPO_LN_BWD");
    v = (e && atoi(e) == 1) ? 0 : 1;
  }
  return v == 1;
}

int ppo_layernorm_bwd(const void* x, const float* gamma, const void* dy, const void* resid_grad, void* dx,
                      float* dgamma, float* dbeta, int64_t rows, int64_t hidden, float eps, void* drop_out, float p,
                      uint64_t drop_seed, uint64_t drop_offset, const uint64_t* drop_offset_base, const float* beta,
                      void* ln_out, void* stream) {
  if (int rc = check_rows("ppo_layernorm_bwd", rows, hidden)) return rc;
  if (!x || !gamma || !dy || !dx || !dgamma || !dbeta) return set_error(PPO_EINVAL, "ppo_layernorm_bwd: null pointer");
  if (ln_out && !beta) return set_error(PPO_EINVAL, "ppo_layernorm_bwd: ln_out needs beta");
  if (!(p >= 0.f && p < 1.f)) return set_error(PPO_EINVAL, "ppo_layernorm_bwd: p=%f", p);
  if (rows == 0) return PPO_OK;
  RowLaunch l;
  int rc = PPO_OK;
  if (!aligned16(dgamma) || !aligned16(dbeta) || !aligned16(gamma) || (beta && !aligned16(beta)))
    return set_error(PPO_EINVAL, "ppo_layernorm_bwd: gamma/beta/dgamma/dbeta must be 16-byte aligned");
  // Two vectors per lane per tensor: W = h/512 warps per row (up to 16 at h = 8192).
  const int need = warps_per_row(hidden, 2);
#define PPO_LN_BWD_K(W, O, P)                                                                                  \
  {                                                                                                            \
    constexpr int G = groups_for(W);                                                                           \
    if ((rc = row_launch(ln_bwd_kernel<W, 2, G, O, P>, rows, hidden, W, 2, &l, G))) return rc;                \
    launch_pdl(ln_bwd_kernel<W, 2, G, O, P>, l.grid, l.block, l.smem, as_stream(stream),                       \
        static_cast<const __nv_bfloat16*>(x), gamma, beta, static_cast<const __nv_bfloat16*>(dy),             \
        static_cast<const __nv_bfloat16*>(resid_grad), static_cast<__nv_bfloat16*>(dx), dgamma, dbeta,        \
        static_cast<__nv_bfloat16*>(ln_out), rows, (int)hidden, eps, static_cast<__nv_bfloat16*>(drop_out),   \
        dropout_threshold(p), p > 0.f ? 1.f / (1.f - p) : 1.f, drop_seed, drop_offset, drop_offset_base);     \
  }
#define PPO_LN_BWD_W(W)                                            \
  {                                                                \
    /* with the LN recompute output the prefetching kernel spills at */ \
    /* W <= 5 (2 words): no prefetch there (C2: 30.8 vs 37.0 us)      */ \
    const bool pf = ln_bwd_prefetch() && !(ln_out && W <= 5);      \
    if (ln_out) {                                                  \
      if (pf) PPO_LN_BWD_K(W, true, true) else PPO_LN_BWD_K(W, true, false) \
    } else {                                                       \
      if (pf) PPO_LN_BWD_K(W, false, true) else PPO_LN_BWD_K(W, false, false) \
    }                                                              \
  }
  if (need <= 1) PPO_LN_BWD_W(1)
  else if (need <= 2) PPO_LN_BWD_W(2)
  else if (need <= 3) PPO_LN_BWD_W(3)
  else if (need <= 4) PPO_LN_BWD_W(4)
  else if (need <= 5) PPO_LN_BWD_W(5)
  else if (need <= 6) PPO_LN_BWD_W(6)
  else if (need <= 8) PPO_LN_BWD_W(8)
  else if (need <= 10) PPO_LN_BWD_W(10)
  else if (need <= 12) PPO_LN_BWD_W(12)
  else PPO_LN_BWD_W(16)
#undef PPO_LN_BWD_W
#undef PPO_LN_BWD_K
  PPO_LAUNCHED("ln_bwd_kernel");
  return PPO_OK;
}

int ppo_layernorm_fwd2(const void* x_a, const float* gamma_a, const float* beta_a, void* y_a, const void* x_b,
                       const float* gamma_b, const float* beta_b, void* y_b, int64_t rows, int64_t hidden, float eps,
                       void* stream) {
  if (int rc = check_rows("ppo_layernorm_fwd2", rows, hidden)) return rc;
  if (!x_a || !gamma_a || !beta_a || !y_a || !x_b || !gamma_b || !beta_b || !y_b)
    return set_error(PPO_EINVAL, "ppo_layernorm_fwd2: null pointer");
  if (rows == 0) return PPO_OK;
  RowLaunch l;
  int rc = PPO_OK;
  const int vpl = vpl_choice(hidden, 4);
#define PPO_LN_FWD2_W(W, V)                                                                                   \
  if ((rc = row_launch(ln_fwd_kernel<false, W, V, fwd_groups_for(W), true>, 2 * rows, hidden, W, 0, &l,       \
                       fwd_groups_for(W)))) return rc;                                                        \
  launch_pdl(ln_fwd_kernel<false, W, V, fwd_groups_for(W), true>, l.grid, l.block, l.smem, as_stream(stream),  \
      static_cast<const __nv_bfloat16*>(x_b), static_cast<const __nv_bfloat16*>(x_a),                        \
      static_cast<__nv_bfloat16*>(y_b), gamma_a, beta_a, static_cast<__nv_bfloat16*>(y_a), 2 * rows,          \
      (int)hidden, eps, 0u, 1.f, (uint64_t)0, (uint64_t)0, (const uint64_t*)nullptr, 0, gamma_b, beta_b, rows);
#define PPO_LN_FWD2_V(V)                                              \
  {                                                                   \
    switch (warps_per_row(hidden, V)) {                               \
      case 1: PPO_LN_FWD2_W(1, V) break;                              \
      case 2: PPO_LN_FWD2_W(2, V) break;                              \
      case 3: PPO_LN_FWD2_W(3, V) break;                              \
      case 4: PPO_LN_FWD2_W(4, V) break;                              \
      case 5: PPO_LN_FWD2_W(5, V) break;                              \
      case 6: PPO_LN_FWD2_W(6, V) break;                              \
      case 7: PPO_LN_FWD2_W(7, V) break;                              \
      default: PPO_LN_FWD2_W(8, V) break;                             \
    }                                                                 \
  }
  PPO_VPL_DISPATCH(vpl, PPO_LN_FWD2_V)
#undef PPO_LN_FWD2_V
#undef PPO_LN_FWD2_W
  PPO_LAUNCHED("ln_fwd_kernel<dual>");
  return PPO_OK;
}

}  // extern "C"
