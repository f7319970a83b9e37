// libppo_b200.so -- K7 causal attention forward, hand-written on tcgen05 (sm_100a).
//
// o[s, h] (bf16, written straight into the activation slab) and lse[heads, s] (fp32,
// natural log -- the statistics K7b and cuDNN's backward consume) from the fused
// qkv[s, 3h] of one microbatch.  The reference holds only the FLOP model of this op
// (pkg/src/ppoff/costs.py:144-161: 12bs^2h of the 12bsh(6h+s) per layer) and keeps o and
// the softmax statistics in the saved set it prices (costs.py:99-105).
//
// One CTA per (pair of adjacent 128-row q blocks i0 = 2t, i1 = 2t + 1, head): q block i0
// walks kv blocks 0..i0, i1 walks 0..i1; every K/V tile is loaded once by TMA for both.
// Per (q block, kv block): S = Q K^T (A = Q, B = K, both K-major shared memory) into
// TMEM, the softmax warpgroup of that q block (one thread per q row, the row in
// registers) turns S into P = exp2(S * scale * log2e - m) with a running row maximum m
// that is only moved when it grows by more than 2^8 (O is rescaled in TMEM then, rarely
// after the first kv blocks), writes P as bf16 over S's first 64 TMEM columns, and
// O += P V runs with A = P from TMEM and B = V (MN-major shared memory).  The two q blocks
// ping-pong: the tensor core runs S/PV of one while the other's warpgroup exponentiates.
// TMEM: S0 [0,128), S1 [128,256), O0 [256, 256+D), O1 [256+D, 256+2D).
// Warps: 0-3 softmax of q block i0, 4-7 of i1, 8 UMMA issue (converged, one lane issues),
// 9 TMA producer, 10-11 register donors (setmaxnreg).
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "ppo_common.cuh"
#include "ppo_tcgen05.cuh"

#ifndef PPO_FWD_POLY
#define PPO_FWD_POLY 1  // measured: 0 / 1 / 2 / 3 / 4 per 8 -> 68.8 / 65.7 / 66.9 / 67.0 / 70.4 us at C2
#endif

namespace ppo {
namespace attnf {

using namespace ppo::tc;

constexpr int kTile = 128;
constexpr int kThreads = 384;

template <int D>
struct Cfg {
  static constexpr int kHalves = D / 64;
  static constexpr int kTileBytes = kHalves * kHalf;
  static constexpr int kOffQ = 0;                      // q0, q1
  static constexpr int kOffKV = 2 * kTileBytes;        // 2 stages x (K, V)
  static constexpr int kOffBar = kOffKV + 4 * kTileBytes;
  static constexpr int kNumBars = 24;
  static constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
  static constexpr int kOffItems = kOffTmemPtr + 16;  // 4 work-item slots
  static constexpr int kSmemBytes = kOffItems + 16;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
  static constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO0 = 256, kColO1 = 256 + D;
};

enum : int {
  B_Q = 0,     // Q of the current item landed
  B_KVF0 = 1,  // kv full[2]
  B_KVE0 = 3,  // kv empty[2]
  B_SF0 = 5,   // S full[2] (q block 0 / 1)
  B_PF0 = 7,   // P full[2]
  B_OD0 = 9,   // O done[2]: the PV of the last issued step has completed
  B_QE = 11,   // Q of the item no longer read (its last S issued and done)
  B_OE0 = 12,  // O[2] read by the item's epilogue: the next item may accumulate
  B_ITEM0 = 14,  // item slot full[4]
};

struct Params {
  __nv_bfloat16* o;
  float* lse;  // [H, s] natural log
  int s, H;
  float scale;
  long long* trace;  // diagnostics: per-event SM clocks of CTA 0's first item, or null
  int head_group;    // heads walked together (dispatch order), divides H
  int* work;         // [2]: work counter, finished CTAs (the last one resets both)
};

// diagnostics (ppo_attn_fwd_trace; compiled in with -DPPO_ATTN_TRACE=1 only -- the probes
// cost ~7% at C2, tools/variant_build.py): event e of step j of work item 0 at trace[e * 256 + j]
#ifndef PPO_ATTN_TRACE
#define PPO_ATTN_TRACE 0
#endif
#define ATF_TRACE(e, j)                                                                          \
  do {                                                                                           \
    if (PPO_ATTN_TRACE && p.trace && trace_item && (j) < 256) p.trace[(e) * 256 + (j)] = clock64(); \
  } while (0)

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const Params p) {
  using C = Cfg<D>;
  constexpr int kTileBytes = C::kTileBytes;
  constexpr int kDK = D / 16;  // UMMA K-steps over the head dimension (S)
  constexpr int kPolyPer8 = PPO_FWD_POLY;  // exponentials per 8 on the FMA pipe, the rest on the SFU
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Persistent: work item w = (q-block pair, head) in dispatch order -- groups of head_group
  // heads, the heaviest pairs first inside a group, heads innermost, so concurrent CTAs share
  // the K / V tiles of a few heads in L2 (C4: 40 heads x 16 MB of K, V) -- taken from a global
  // counter when the CTA's producer gets to it (greedy longest first), handed to the other
  // roles through a 4-slot shared-memory ring.  The next item's Q and first K/V land while
  // the previous item's O leaves.
  const int n_pairs = p.s / (2 * kTile), n_items = p.H * n_pairs;
  auto decode = [&](int w, int& i0, int& hd) {
    const int per_group = p.head_group * n_pairs, grp = w / per_group, rem = w % per_group;
    hd = grp * p.head_group + rem % p.head_group;
    i0 = 2 * (n_pairs - 1 - rem / p.head_group);
  };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::kOffTmemPtr);
  volatile int* item_slot = reinterpret_cast<volatile int*>(smem + C::kOffItems);
  auto next_item = [&](int r) {  // consumers: item of round r, -1 when the CTA is done
    mbar_wait(&bars[B_ITEM0 + (r & 3)], (r >> 2) & 1);
    return item_slot[r & 3];
  };
  bool trace_item = false;

  if (threadIdx.x == 0) {
    mbar_init(&bars[B_Q], 1);
    mbar_init(&bars[B_QE], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars[B_KVF0 + i], 1);
      mbar_init(&bars[B_KVE0 + i], 1);
      mbar_init(&bars[B_SF0 + i], 1);
      mbar_init(&bars[B_PF0 + i], 4);
      mbar_init(&bars[B_OD0 + i], 1);
      mbar_init(&bars[B_OE0 + i], 4);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&bars[B_ITEM0 + i], 1);
    mbar_fence_init();
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_ptr))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 9 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_qkv)) : "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  const uint32_t sbase = smem_u32(smem);

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    if (warp == 9) {
      // ===================================================== TMA producer
      if (lane == 0) {
        const int H = p.H;
        int gk = 0;  // kv tiles loaded so far (ring index)
        for (int r = 0;; ++r) {
          int w = atomicAdd(&p.work[0], 1);
          w = w < n_items ? w : -1;
          item_slot[r & 3] = w;
          mbar_arrive(&bars[B_ITEM0 + (r & 3)]);
          if (w < 0) break;
          int i0, hd;
          decode(w, i0, hd);
          mbar_wait(&bars[B_QE], (r & 1) ^ 1);  // the previous item's last S is done
          mbar_expect_tx(&bars[B_Q], 2 * kTileBytes);
          for (int q = 0; q < 2; ++q)
            for (int half = 0; half < C::kHalves; ++half)
              tma_load_3d(smem + C::kOffQ + q * kTileBytes + half * kHalf, &tm_qkv, half * 64, hd,
                          (i0 + q) * kTile, &bars[B_Q]);
          for (int j = 0; j < i0 + 2; ++j, ++gk) {
            const int st = gk & 1;
            mbar_wait(&bars[B_KVE0 + st], ((gk >> 1) & 1) ^ 1);
            mbar_expect_tx(&bars[B_KVF0 + st], 2 * kTileBytes);
            uint8_t* kv = smem + C::kOffKV + st * 2 * kTileBytes;
            for (int half = 0; half < C::kHalves; ++half) {
              tma_load_3d(kv + half * kHalf, &tm_qkv, half * 64, H + hd, j * kTile, &bars[B_KVF0 + st]);
              tma_load_3d(kv + kTileBytes + half * kHalf, &tm_qkv, half * 64, 2 * H + hd, j * kTile,
                          &bars[B_KVF0 + st]);
            }
          }
        }
      }
    } else if (warp == 8) {
      // ===================================================== UMMA issuer (converged warp)
      const uint32_t sb4 = sbase >> 4;
      const uint32_t aQ0 = sb4 + (C::kOffQ >> 4), aQ1 = sb4 + ((C::kOffQ + kTileBytes) >> 4);
      const uint32_t tS0 = tmem + C::kColS0, tS1 = tmem + C::kColS1, tO0 = tmem + C::kColO0,
                     tO1 = tmem + C::kColO1;
      constexpr uint32_t I_S = idesc(0, 0, 128), I_PV = idesc(0, 1, D);
      int gk = 0, g0 = 0, g1 = 0;  // kv tiles, PV steps of q block 0 / 1 (barrier phases)
      auto aK = [&](int k) { return sb4 + ((C::kOffKV + (k & 1) * 2 * kTileBytes) >> 4); };
      auto aV = [&](int k) { return sb4 + ((C::kOffKV + (k & 1) * 2 * kTileBytes + kTileBytes) >> 4); };
      auto kv_wait = [&](int k) { mbar_wait(&bars[B_KVF0 + (k & 1)], (k >> 1) & 1); };
      for (int r = 0, w; (w = next_item(r)) >= 0; ++r) {
        int i0, hd;
        decode(w, i0, hd);
        trace_item = w == 0;
        const int n0 = i0 + 1, n1 = i0 + 2;
        mbar_wait(&bars[B_Q], r & 1);
        kv_wait(gk);
        tc_fence_after();
        gemm128<kDK, false, false, false>(tS0, aQ0, aK(gk), I_S, false);  // S0(0)
        tc_commit(&bars[B_SF0]);
        gemm128<kDK, false, false, false>(tS1, aQ1, aK(gk), I_S, false);  // S1(0)
        tc_commit(&bars[B_SF0 + 1]);
        for (int j = 0; j < n1; ++j) {
          const int k = gk + j;
          ATF_TRACE(0, j);
          if (j < n0) {  // O0 += P0(j) V_j
            mbar_wait(&bars[B_PF0], (g0 + j) & 1);
            ATF_TRACE(1, j);
            if (j == 0 && r > 0) mbar_wait(&bars[B_OE0], (r - 1) & 1);  // previous item's O0 read
            tc_fence_after();
            gemm128<8, false, true, true>(tO0, tS0, aV(k), I_PV, j > 0);
            tc_commit(&bars[B_OD0]);
          }
          if (j + 1 < n0) {  // S0(j+1): P0(j) in the same columns was read by the PV just issued
            kv_wait(k + 1);
            tc_fence_after();
            gemm128<kDK, false, false, false>(tS0, aQ0, aK(k + 1), I_S, false);
            tc_commit(&bars[B_SF0]);
          }
          ATF_TRACE(2, j);
          mbar_wait(&bars[B_PF0 + 1], (g1 + j) & 1);  // O1 += P1(j) V_j
          ATF_TRACE(3, j);
          if (j == 0 && r > 0) mbar_wait(&bars[B_OE0 + 1], (r - 1) & 1);
          tc_fence_after();
          gemm128<8, false, true, true>(tO1, tS1, aV(k), I_PV, j > 0);
          tc_commit(&bars[B_OD0 + 1]);
          tc_commit(&bars[B_KVE0 + (k & 1)]);  // K_j, V_j consumed
          if (j + 1 < n1) {
            kv_wait(k + 1);
            tc_fence_after();
            gemm128<kDK, false, false, false>(tS1, aQ1, aK(k + 1), I_S, false);
            tc_commit(&bars[B_SF0 + 1]);
          } else {
            tc_commit(&bars[B_QE]);  // every S of the item issued: Q may be replaced
          }
        }
        gk += n1;
        g0 += n0;
        g1 += n1;
      }
    }
    // warps 10, 11: idle register donors
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    // ===================================================== softmax warpgroups
    const int wg = warp >> 2, quarter = warp & 3;
    const int row = quarter * 32 + lane;  // q row within the block (TMEM lane)
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_off + (wg ? C::kColS1 : C::kColS0);
    const uint32_t tO = tmem + lane_off + (wg ? C::kColO1 : C::kColO0);
    const float sl2 = p.scale * 1.4426950408889634f;
    int gs = 0;  // steps of this q block in earlier items (barrier phases)
    for (int r = 0, w; (w = next_item(r)) >= 0; ++r) {
      int i0, hd;
      decode(w, i0, hd);
      trace_item = w == 0;
      const int qi = i0 + wg, nk = qi + 1;
      float m = -INFINITY, l = 0.f;  // running max (log2 domain, already scaled) and sum
      for (int j = 0; j < nk; ++j) {
        const int gj = gs + j;
        mbar_wait(&bars[B_SF0 + wg], gj & 1);
        if (quarter == 0 && lane == 0) ATF_TRACE(10 + 4 * wg, j);
        tc_fence_after();
        uint32_t rr[4][32];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) tmem_ld32(tS + ch * 32, rr[ch]);
        tmem_wait_ld();
        if (quarter == 0 && lane == 0) ATF_TRACE(13 + 4 * wg, j);
        if (j == qi) {  // the diagonal block: kv column c > q row is masked
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c > row) rr[c >> 5][c & 31] = __float_as_uint(-INFINITY);
        }
        float mx;
        {
          float a0 = -INFINITY, a1 = -INFINITY, a2 = -INFINITY, a3 = -INFINITY;
#pragma unroll
          for (int c = 0; c < 128; c += 8) {
            a0 = fmax3(a0, __uint_as_float(rr[c >> 5][c & 31]), __uint_as_float(rr[c >> 5][(c + 1) & 31]));
            a1 = fmax3(a1, __uint_as_float(rr[c >> 5][(c + 2) & 31]), __uint_as_float(rr[c >> 5][(c + 3) & 31]));
            a2 = fmax3(a2, __uint_as_float(rr[c >> 5][(c + 4) & 31]), __uint_as_float(rr[c >> 5][(c + 5) & 31]));
            a3 = fmax3(a3, __uint_as_float(rr[c >> 5][(c + 6) & 31]), __uint_as_float(rr[c >> 5][(c + 7) & 31]));
          }
          mx = fmax3(a0, a1, fmaxf(a2, a3));
        }
        const float m_new = fmaxf(m, mx * sl2);
        if (quarter == 0 && lane == 0) ATF_TRACE(20 + wg, j);
        if (quarter == 0 && lane == 0) ATF_TRACE(20 + wg, j);
        // move the maximum only when it grows by more than 8 (P stays <= 2^8 otherwise)
        const bool move = m_new > m + 8.f;
        const float alpha = move ? ex2(m - m_new) : 1.f;
        if (move) m = m_new;
        // x = s * scale * log2e - m on packed pairs; a share of the exponentials on the FMA
        // pipe (not in the diagonal step, whose masked -inf scores go through the SFU)
        const uint64_t sl2x2 = f2(sl2, sl2), nm2 = f2(-m, -m);
        uint64_t sum2 = f2(0.f, 0.f);
        uint32_t pk[64];
        auto exps = [&](auto poly) {  // poly: std::true_type off the diagonal
#pragma unroll
          for (int c = 0; c < 128; c += 2) {
            const float2 x = f2u(ffma2(f2(__uint_as_float(rr[c >> 5][c & 31]), __uint_as_float(rr[c >> 5][(c + 1) & 31])),
                                       sl2x2, nm2));
            float2 e;
            if (decltype(poly)::value && (c & 7) < 2 * (kPolyPer8 / 2)) {
              e = ex2_fma2(x.x, x.y);
            } else if (decltype(poly)::value && (c & 7) == 2 * (kPolyPer8 / 2) && (kPolyPer8 & 1)) {
              e = make_float2(ex2_fma(x.x), ex2(x.y));
            } else {
              e = make_float2(ex2(x.x), ex2(x.y));
            }
            sum2 = fadd2(sum2, f2(e.x, e.y));
            pk[c >> 1] = pack_bf16(e.x, e.y);
          }
        };
        if (j == qi) exps(std::false_type{});  // masked -inf scores go through the SFU
        else exps(std::true_type{});
        const float2 sp = f2u(sum2);
        l = l * alpha + (sp.x + sp.y);
        if (quarter == 0 && lane == 0) ATF_TRACE(11 + 4 * wg, j);
        if (lane == 0) ATF_TRACE(24 + 4 * wg + quarter, j);  // exponentials done, per warp
        // O rescale (rows whose maximum moved) once the previous PV of this block is done
        if (j > 0 && __any_sync(0xffffffffu, move)) {
          mbar_wait(&bars[B_OD0 + wg], (gj - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int ch = 0; ch < D / 32; ++ch) {
            uint32_t o[32];
            tmem_ld32(tO + ch * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
            tmem_st32(tO + ch * 32, o);
          }
        }
        {
          uint32_t (&p0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&pk[0]);
          uint32_t (&p1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&pk[32]);
          tmem_st32(tS, p0);
          tmem_st32(tS + 32, p1);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_PF0 + wg]);
        if (quarter == 0 && lane == 0) ATF_TRACE(12 + 4 * wg, j);
      }
      gs += nk;
      // ---- epilogue: o = O / l (bf16) into the slab, lse = ln 2 * (m + log2 l)
      mbar_wait(&bars[B_OD0 + wg], (gs - 1) & 1);
      tc_fence_after();
      uint32_t ov[D];
#pragma unroll
      for (int ch = 0; ch < D / 32; ++ch) tmem_ld32(tO + ch * 32, *reinterpret_cast<uint32_t(*)[32]>(&ov[ch * 32]));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_OE0 + wg]);  // the next item may accumulate into O
      const float inv = 1.f / l;
      const size_t h = size_t(p.H) * D;
      const size_t q = size_t(qi) * kTile + row;
      __nv_bfloat16* dst = p.o + q * h + size_t(hd) * D;
#pragma unroll
      for (int v = 0; v < D / 8; ++v) {
        uint4 wq;
        wq.x = pack_bf16(__uint_as_float(ov[8 * v + 0]) * inv, __uint_as_float(ov[8 * v + 1]) * inv);
        wq.y = pack_bf16(__uint_as_float(ov[8 * v + 2]) * inv, __uint_as_float(ov[8 * v + 3]) * inv);
        wq.z = pack_bf16(__uint_as_float(ov[8 * v + 4]) * inv, __uint_as_float(ov[8 * v + 5]) * inv);
        wq.w = pack_bf16(__uint_as_float(ov[8 * v + 6]) * inv, __uint_as_float(ov[8 * v + 7]) * inv);
        *reinterpret_cast<uint4*>(dst + v * 8) = wq;
      }
      p.lse[size_t(hd) * p.s + q] = (m + __log2f(l)) * 0.69314718055994530942f;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  if (threadIdx.x == 0) {  // the last CTA out resets the work counter for the next launch
    __threadfence();
    if (atomicAdd(&p.work[1], 1) == int(gridDim.x) - 1) {
      p.work[0] = 0;
      p.work[1] = 0;
      __threadfence();
    }
  }
}

long long* g_trace = nullptr;

// Work counters: a ring of 8192 zeroed pairs per device, created on the first call (which
// must not be inside a stream capture -- Stage._attn_init makes one eagerly); a launch takes
// the next pair and its last CTA resets it, so launches in flight on different streams
// (ranks sharing a GPU, each replaying graphs with up to a few hundred launches) never
// share a counter.
constexpr unsigned kWorkSlots = 8192;

static int* work_slot(int* rc) {
  static std::mutex mu;
  static int* bufs[64] = {};
  static unsigned next[64] = {};
  *rc = PPO_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) {
    *rc = set_error(PPO_EINVAL, "ppo_attn_fwd: device %d", dev);
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (!bufs[dev]) {
    int* d = nullptr;
    cudaError_t e = cudaMalloc(&d, kWorkSlots * 2 * sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(d, 0, kWorkSlots * 2 * sizeof(int));
    if (e != cudaSuccess) {
      *rc = cuda_error(e, "ppo_attn_fwd: work counters (the first call must not be inside a stream capture)");
      return nullptr;
    }
    bufs[dev] = d;
  }
  return bufs[dev] + 2 * (next[dev]++ % kWorkSlots);
}

template <typename K>
static int smem_optin(K kernel, int bytes, unsigned* done) {
  static std::mutex mu;
  int dev = 0;
  PPO_TRY_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 32 && (*done >> dev) & 1u) return PPO_OK;
  PPO_TRY_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  if (dev < 32) *done |= 1u << dev;
  return PPO_OK;
}

template <int D>
static int launch(const CUtensorMap& tm, const Params& prm, dim3 grid, cudaStream_t st) {
  static unsigned done = 0;
  int rc;
  if ((rc = smem_optin(attn_fwd_kernel<D>, Cfg<D>::kSmemBytes, &done))) return rc;
  attn_fwd_kernel<D><<<grid, kThreads, Cfg<D>::kSmemBytes, st>>>(tm, prm);
  return PPO_OK;
}

}  // namespace attnf

// Hand-written forward (used by ppo_attn_fwd, ppo_attention.cu).  seq % 256 == 0,
// head_dim 64 / 128, arguments validated by the caller.
int attn_fwd_tcgen05(const void* qkv, void* o, float* lse, int s, int H, int D, float scale, cudaStream_t st) {
  using namespace attnf;
  int rc = PPO_OK;
  tc::EncodeTiled enc = tc::encoder(&rc);
  if (rc) return rc;
  const int64_t h = int64_t(H) * D;
  CUtensorMap tm;
  if ((rc = tc::make_map(enc, &tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, qkv, D, 3 * H, s, 3 * h * 2, 64, kTile)))
    return rc;
  static const int group_env = [] {
    const char* e = std::getenv("PPO_ATTN_HEAD_GROUP");  // A/B experiments
    return e ? std::atoi(e) : 0;
  }();
  // group heads only when one operand pair of all heads (4 s h bytes) outgrows a half of L2;
  // below that the all-heads LPT order packs the SMs better (C2 forward 66 vs 70 us)
  const bool big = 4.0 * double(s) * double(H) * double(D) > 64.0 * (1 << 20);
  int group = group_env > 0 ? group_env : (big ? 8 : H);
  while (H % group) --group;
  int* work = work_slot(&rc);
  if (rc) return rc;
  Params prm{static_cast<__nv_bfloat16*>(o), lse, s, H, scale, attnf::g_trace, group, work};
  const int items = H * (s / (2 * kTile)), sms = sm_count_current();
  const dim3 grid(items < sms ? items : sms);
  if ((rc = D == 64 ? launch<64>(tm, prm, grid, st) : launch<128>(tm, prm, grid, st))) return rc;
  PPO_LAUNCHED("attn_fwd_kernel");
  return PPO_OK;
}

}  // namespace ppo

extern "C" int ppo_attn_fwd_trace(void* trace) {
  ppo::attnf::g_trace = static_cast<long long*>(trace);
  return PPO_OK;
}
