// libppo_b200.so -- K7b causal attention backward on tcgen05 (sm_100a), hand-written.
//
//   ppo_attn_bwd   dqkv[s, 3h] (bf16: dq | dk | dv, the layout the QKV projection's
//                  dgrad and wgrad GEMMs consume as one operand) from qkv[s, 3h], the
//                  saved o[s, h] and lse[heads, s] (both reloaded from the activation
//                  slab), and the output gradient do[s, h].
//
// The reference prices attention only through its FLOP model (pkg/src/ppoff/costs.py:
// 144-161: the s-term of 12bsh(6h+s), backward = 2x forward) and keeps o and the softmax
// statistics in the saved set (costs.py:99-105), so the backward needs no recompute of
// the forward statistics: P = exp(scale * Q K^T - lse).
//
// Persistent: one CTA per SM takes work items (kv block j of 128 rows, head) from a global
// counter, longest walks first; an item walks the q blocks i >= j (causal) and keeps dK_j,
// dV_j in TMEM for the whole walk, then stores them by TMA while the next item's K_j, V_j
// land.  Per (i, j) tile, five 128x128x(16k) UMMAs
// (tcgen05.mma.cta_group::1.kind::f16, fp32 accumulators in TMEM):
//
//   S^T  = K_j Q_i^T           A = K  smem K-major   B = Q  smem K-major   -> TMEM S
//   dP^T = V_j dO_i^T          A = V  smem K-major   B = dO smem K-major   -> TMEM dP
//   dV  += P^T dO_i            A = P^T TMEM (bf16)   B = dO smem MN-major  -> TMEM dV
//   dK  += dS^T Q_i            A = dS^T smem K-major B = Q  smem MN-major  -> TMEM dK
//   dQ_i = dS K_j              A = dS smem MN-major  B = K  smem MN-major  -> TMEM dQ (= dP cols)
//
// Issue order per step i (one thread): S(i); dK(i-1), dQ(i-1) once dS(i-1) is in shared
// memory; dP(i) once the drain warps hold dQ(i-1); dV(i) once P(i) is in TMEM.  The
// softmax-gradient warps of step i overlap the tensor core's dK/dQ of step i-1.
//
// Every operand tile is loaded once by TMA in the 128-byte-swizzled layout and read by
// the tensor core both K-major and MN-major (the swizzle atom of 8 rows x 128 B is the
// same physical arrangement for both), so Q, dO and K feed two UMMAs each without a
// transpose.  dQ partials leave through TMA bulk reduce-add (cp.reduce.async.bulk.tensor
// .add.f32) into an fp32 accumulator; a small kernel scales and casts it into dqkv (a
// fused cast by the last contributor per block was measured: waiting for the reduce-adds
// to complete takes ~20000 clocks, the cast stays a kernel of its own).
//
// Warp roles (512 threads): warps 0-3 drain dQ from TMEM into the reduce-add, warps 4-11
// (two warpgroups, q columns 0-63 / 64-127) compute P = exp2(S*scale*log2e - lse*log2e)
// and dS = P (dP - delta), write P^T to TMEM and dS^T to shared memory and run the dK/dV
// epilogue, warp 12 issues the UMMAs (one thread) and owns the TMEM allocation, warp 13
// fetches work items and issues the TMA loads, warps 14-15 donate registers.
// TMEM (512 columns x 128 lanes, D = 128): dK [0,128), dV [128,256), dP / dQ [256,384),
// S [384,512) with P^T (bf16 pairs) over S's first 64 columns (D = 64: Cfg<64>).
#include <cuda.h>  // CUtensorMap; the encoder comes from cudaGetDriverEntryPoint

#include <cstdlib>
#include <mutex>

#include "ppo_common.cuh"
#include "ppo_tcgen05.cuh"

namespace ppo {
namespace attnb {

using namespace ppo::tc;

constexpr int kTile = 128;           // kv rows per CTA, q rows per step
constexpr int kStgBytes = 32 * 32 * 4;

// Per head_dim D (64 or 128): tiles of 128 rows x D are D/64 boxes of 64 columns.
// Shared memory map (bytes from the 1024-aligned dynamic base) and TMEM columns:
// dK [0, D), dV [D, 2D), dP / dQ [2D, 2D + 128), S [2D + 128, 2D + 256) (P^T over its
// first 64 columns).
template <int D>
struct Cfg {
  static constexpr int kHalves = D / 64;
  static constexpr int kTileBytes = kHalves * kHalf;
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + kTileBytes;
  static constexpr int kOffQ = kOffV + kTileBytes;       // 2 stages
  static constexpr int kOffDO = kOffQ + 2 * kTileBytes;  // 1 stage
  static constexpr int kOffDS = kOffDO + kTileBytes;     // 128 x 128 bf16
  static constexpr int kOffStg = kOffDS + 2 * kHalf;     // dQ staging: 4 warps x 2 x 4 KB
  static constexpr int kOffLse = kOffStg + 4 * 2 * kStgBytes;  // 2 stages x 128 fp32
  static constexpr int kOffDelta = kOffLse + 2 * 512;
  static constexpr int kOffBar = kOffDelta + 2 * 512;
  static constexpr int kNumBars = 24;
  static constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
  static constexpr int kOffItems = kOffTmemPtr + 16;  // 4 work-item slots
  static constexpr int kSmemBytes = kOffItems + 16;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
  static constexpr uint32_t kColDK = 0, kColDV = D, kColDP = 2 * D, kColS = 2 * D + 128;
};

// barrier indices
enum : int {
  B_KV = 0,    // K, V of the current item landed
  B_QF0 = 1,   // q_full[2]
  B_QE0 = 3,   // q_empty[2]
  B_DOF = 5,
  B_DOE = 6,
  B_SF = 7,
  B_PF = 8,
  B_DPF = 9,
  B_DSF = 10,
  B_DSE = 11,
  B_DQF = 12,
  B_DQE = 13,
  B_DKV = 14,  // dK, dV of the item complete (and every UMMA of the item)
  B_KVE = 15,  // K, V of the item no longer read: the next item's may land
  B_ACC = 16,  // the epilogue holds dK, dV in registers: the next item may accumulate
  B_ITEM0 = 17,  // item slot full[4] (the producer fetched the next work item)
};

constexpr int kThreads = 512;  // warps 14, 15 idle: setmaxnreg works per warpgroup

struct Params {
  __nv_bfloat16* dqkv;
  const float* lse2;   // [H, s] -log2(e) * logsumexp
  const float* delta;  // [H, s] -rowsum(dO * O)
  float* dq_acc;       // [s, h] fp32
  int* work;           // dynamic work counter (zeroed by the prep kernel)
  int s, H;
  float scale;
  long long* trace;  // diagnostics: per-event SM clocks of CTA (0, 0), or null
  int exp_mode;      // diagnostics (PPO_ATB_EXP): bit 0 no dQ reduce (wrong dq), bit 2 timed GEMMs, bit 3 GEMM forms
  int head_group;    // heads walked together (dispatch order below), divides H
};

// diagnostics (ppo_attn_bwd_trace): event e of step `it` at trace[e * 256 + it]
#define ATB_TRACE(e, it)                                                                     \
  do {                                                                                       \
    if (p.trace && trace_item && (it) < 256) p.trace[(e) * 256 + (it)] = clock64();          \
  } while (0)

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dqkv,
                    const Params p) {
  using C = Cfg<D>;
  constexpr int kTileBytes = C::kTileBytes, kOffK = C::kOffK, kOffV = C::kOffV, kOffQ = C::kOffQ, kOffDO = C::kOffDO,
                kOffDS = C::kOffDS, kOffStg = C::kOffStg, kOffLse = C::kOffLse, kOffDelta = C::kOffDelta,
                kOffBar = C::kOffBar, kOffTmemPtr = C::kOffTmemPtr;
  constexpr uint32_t kColDK = C::kColDK, kColDV = C::kColDV, kColDP = C::kColDP, kColS = C::kColS;
  constexpr int kDK = D / 16;  // UMMA K-steps over the head dimension
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_q = p.s / kTile;
  // Persistent: work item w = (kv block jb, head hd) in dispatch order -- groups of
  // head_group heads, kv block ascending (longest walk first) inside a group, heads
  // innermost, so concurrent CTAs share the Q / dO tiles of a few heads in L2 -- taken from a
  // global counter as a CTA's producer gets to it (a greedy longest-first schedule, like the
  // hardware's in-order dispatch), handed to the other roles through a 4-slot ring in shared
  // memory.  An item's K/V land while the previous item's dK/dV leave.
  const int n_items = p.H * n_q, b = int(blockIdx.x);
  volatile int* item_slot = reinterpret_cast<volatile int*>(smem + C::kOffItems);
  auto next_item = [&](int r) {  // consumers: item of round r, -1 when the CTA is done
    mbar_wait(reinterpret_cast<uint64_t*>(smem + C::kOffBar) + B_ITEM0 + (r & 3), (r >> 2) & 1);
    return item_slot[r & 3];
  };
  auto decode = [&](int w, int& jb, int& hd) {
    const int per_group = p.head_group * n_q, grp = w / per_group, rem = w % per_group;
    jb = rem / p.head_group;
    hd = grp * p.head_group + rem % p.head_group;
  };
  bool trace_item = false;  // diagnostics: events of CTA 0's first item only
  long long* cta_log = p.trace ? p.trace + 64 * 256 + 4 * size_t(b) : nullptr;
  if (cta_log && threadIdx.x == 0) {  // diagnostics: CTA residency (globaltimer ns, SM id, q steps)
    long long t;
    unsigned sm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    cta_log[0] = t;
    cta_log[2] = sm;
  }
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + kOffTmemPtr);
  float* s_lse = reinterpret_cast<float*>(smem + kOffLse);
  float* s_delta = reinterpret_cast<float*>(smem + kOffDelta);

  if (threadIdx.x == 0) {
    mbar_init(&bars[B_KV], 1);
    mbar_init(&bars[B_QF0], 1);
    mbar_init(&bars[B_QF0 + 1], 1);
    mbar_init(&bars[B_QE0], 1);
    mbar_init(&bars[B_QE0 + 1], 1);
    mbar_init(&bars[B_DOF], 1);
    mbar_init(&bars[B_DOE], 1);
    mbar_init(&bars[B_SF], 1);
    mbar_init(&bars[B_PF], 8);
    mbar_init(&bars[B_DPF], 1);
    mbar_init(&bars[B_DSF], 8);
    mbar_init(&bars[B_DSE], 1);
    mbar_init(&bars[B_DQF], 1);
    mbar_init(&bars[B_DQE], 4);
    mbar_init(&bars[B_DKV], 1);
    mbar_init(&bars[B_KVE], 1);
    mbar_init(&bars[B_ACC], 8);
    for (int i = 0; i < 4; ++i) mbar_init(&bars[B_ITEM0 + i], 1);
    mbar_fence_init();
  }
  if (warp == 12) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_ptr))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 13 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_qkv)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_do)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_dq)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_dqkv)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  const uint32_t sbase = smem_u32(smem);
  // register budget per warpgroup (64K registers / 512 threads = 128 at launch): the
  // issue warpgroup (12-15) gives 72 per thread to the dQ drain and softmax-gradient
  // warpgroups (152 each).  Each side's roles branch below without re-merging, so the
  // allocator sees one budget per path.
  if (warp >= 12) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");

  if (warp == 13) {
    // ===================================================== TMA producer
    if (lane == 0) {
      const int H = p.H;
      int g = 0;  // q steps of earlier items (global step index base)
      for (int r = 0;; ++r) {
        int w = atomicAdd(p.work, 1);
        w = w < n_items ? w : -1;
        item_slot[r & 3] = w;
        mbar_arrive(&bars[B_ITEM0 + (r & 3)]);  // release: the slot write is visible to waiters
        if (w < 0) break;
        int jb, hd;
        decode(w, jb, hd);
        trace_item = b == 0 && r == 0;
        const int n_it = n_q - jb;
        auto load_step = [&](int it) {
          const int gi = g + it, qb = jb + it, st = gi & 1;
          mbar_wait(&bars[B_QE0 + st], ((gi >> 1) & 1) ^ 1);
          ATB_TRACE(28, it);
          mbar_expect_tx(&bars[B_QF0 + st], kTileBytes + 1024);
          for (int half = 0; half < C::kHalves; ++half)
            tma_load_3d(smem + kOffQ + st * kTileBytes + half * kHalf, &tm_qkv, half * 64, hd, qb * kTile,
                        &bars[B_QF0 + st]);
          tma_load_1d(s_lse + st * 128, p.lse2 + size_t(hd) * p.s + qb * kTile, 512, &bars[B_QF0 + st]);
          tma_load_1d(s_delta + st * 128, p.delta + size_t(hd) * p.s + qb * kTile, 512, &bars[B_QF0 + st]);
          mbar_wait(&bars[B_DOE], (gi & 1) ^ 1);
          ATB_TRACE(29, it);
          mbar_expect_tx(&bars[B_DOF], kTileBytes);
          for (int half = 0; half < C::kHalves; ++half)
            tma_load_3d(smem + kOffDO + half * kHalf, &tm_do, half * 64, hd, qb * kTile, &bars[B_DOF]);
        };
        load_step(0);  // the first Q / dO of this item may land before its K / V
        mbar_wait(&bars[B_KVE], (r & 1) ^ 1);
        mbar_expect_tx(&bars[B_KV], 2 * kTileBytes);
        for (int half = 0; half < C::kHalves; ++half) {
          tma_load_3d(smem + kOffK + half * kHalf, &tm_qkv, half * 64, H + hd, jb * kTile, &bars[B_KV]);
          tma_load_3d(smem + kOffV + half * kHalf, &tm_qkv, half * 64, 2 * H + hd, jb * kTile, &bars[B_KV]);
        }
        for (int it = 1; it < n_it; ++it) load_step(it);
        g += n_it;
      }
      if (cta_log) cta_log[3] = g;  // q steps this CTA walked
    }
  } else if (warp == 12) {
    // ===================================================== UMMA issuer (converged warp, one lane issues)
    const uint32_t sb4 = sbase >> 4;
    const uint32_t aK = sb4 + (kOffK >> 4), aV = sb4 + (kOffV >> 4), aDO = sb4 + (kOffDO >> 4),
                   aDS = sb4 + (kOffDS >> 4);
    const uint32_t tS = tmem + kColS, tDP = tmem + kColDP, tDV = tmem + kColDV, tDK = tmem + kColDK;
    constexpr uint32_t I_KK = idesc(0, 0), I_KMd = idesc(0, 1, D), I_MMd = idesc(1, 1, D);
    int g = 0;
    for (int r = 0, w; (w = next_item(r)) >= 0; ++r) {
      int jb, hd;
      decode(w, jb, hd);
      trace_item = b == 0 && r == 0;
      const int n_it = n_q - jb;
      mbar_wait(&bars[B_KV], r & 1);
      tc_fence_after();
      for (int it = 0; it <= n_it; ++it) {
        const int gi = g + it, st = gi & 1;
        const uint32_t aQ = sb4 + ((kOffQ + st * kTileBytes) >> 4);
        if (it < n_it) {
          mbar_wait(&bars[B_QF0 + st], (gi >> 1) & 1);
          ATB_TRACE(0, it);
          tc_fence_after();
          gemm128<kDK, false, false, false>(tS, aK, aQ, I_KK, false);  // S^T = K Q^T
          tc_commit(&bars[B_SF]);
          ATB_TRACE(1, it);
        }
        if (it > 0) {
          // dK(it-1), dQ(it-1): dS(it-1) is in shared memory.  dK first: its Q stage goes
          // back to the producer one GEMM earlier (period 3839 vs 4128 clocks at C2)
          const int pt = it - 1, gp = gi - 1;
          const uint32_t aQp = sb4 + ((kOffQ + (gp & 1) * kTileBytes) >> 4);
          mbar_wait(&bars[B_DSF], gp & 1);
          ATB_TRACE(2, pt);
          tc_fence_after();
          gemm128<8, false, true, false>(tDK, aDS, aQp, I_KMd, pt > 0);  // dK += dS^T Q
          tc_commit(&bars[B_QE0 + (gp & 1)]);
          gemm128<8, true, true, false>(tDP, aDS, aK, I_MMd, false);  // dQ = dS K
          tc_commit(&bars[B_DQF]);
          tc_commit(&bars[B_DSE]);
          ATB_TRACE(3, pt);
          if (it == n_it) {
            tc_commit(&bars[B_DKV]);
            tc_commit(&bars[B_KVE]);
          }
        }
        if (it < n_it) {
          mbar_wait(&bars[B_DOF], gi & 1);
          ATB_TRACE(4, it);
          if (gi > 0) mbar_wait(&bars[B_DQE], (gi - 1) & 1);  // dQ(gi-1) drained: dP reuses its columns
          ATB_TRACE(5, it);
          tc_fence_after();
          gemm128<kDK, false, false, false>(tDP, aV, aDO, I_KK, false);  // dP^T = V dO^T
          tc_commit(&bars[B_DPF]);
          ATB_TRACE(6, it);
          mbar_wait(&bars[B_PF], gi & 1);
          ATB_TRACE(7, it);
          // the previous item's epilogue holds its dK / dV: the accumulators are free
          if (it == 0 && r > 0) mbar_wait(&bars[B_ACC], (r - 1) & 1);
          tc_fence_after();
          gemm128<8, false, true, true>(tDV, tS, aDO, I_KMd, it > 0);  // dV += P^T dO
          tc_commit(&bars[B_DOE]);
          ATB_TRACE(8, it);
        }
      }
      g += n_it;
    }
  }  // warps 14, 15: idle register donors
  } else {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 152;");
  if (warp >= 4) {
    // ===================================================== softmax-gradient warpgroups
    const int wg = (warp - 4) >> 2, quarter = warp & 3;
    const int row = quarter * 32 + lane;  // kv row within the tile (TMEM lane)
    const int c0 = wg * 64;               // q columns of this warpgroup
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const float sl2 = p.scale * 1.4426950408889634f;
    uint8_t* ds_row = smem + kOffDS + wg * kHalf + row * 128;
    int g = 0;
    for (int r = 0, w; (w = next_item(r)) >= 0; ++r) {
      int jb, hd;
      decode(w, jb, hd);
      trace_item = b == 0 && r == 0;
      const int n_it = n_q - jb;
      for (int it = 0; it < n_it; ++it) {
        const int gi = g + it, st = gi & 1;
        const float* lse = s_lse + st * 128 + c0;
        const float* dlt = s_delta + st * 128 + c0;
        mbar_wait(&bars[B_QF0 + st], (gi >> 1) & 1);
        mbar_wait(&bars[B_SF], gi & 1);
        if (warp == 4 && lane == 0) ATB_TRACE(10, it);
        tc_fence_after();
        float pr[64];
        {
          uint32_t rr[2][32];
          tmem_ld32(tmem + lane_off + kColS + c0, rr[0]);
          tmem_ld32(tmem + lane_off + kColS + c0 + 32, rr[1]);
          tmem_wait_ld();
          if (warp == 4 && lane == 0) ATB_TRACE(40, it);
          // x = s * scale * log2e - log2e * lse on packed pairs (s_lse holds -log2e * lse);
          // 1 of 8 exponentials on the FMA pipe (the forward's sweep, ppo_attention_fwd.cu)
          const uint64_t sl2x2 = f2(sl2, sl2);
          const uint64_t* nl = reinterpret_cast<const uint64_t*>(lse);
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            const float2 x = f2u(ffma2(f2(__uint_as_float(rr[c >> 5][c & 31]), __uint_as_float(rr[c >> 5][(c + 1) & 31])),
                                       sl2x2, nl[c >> 1]));
            pr[c] = (c & 7) == 0 ? ex2_fma(x.x) : ex2(x.x);
            pr[c + 1] = ex2(x.y);
          }
        }
        if (it == 0) {  // the diagonal tile: q < kv is masked
#pragma unroll
          for (int c = 0; c < 64; ++c) pr[c] = c0 + c < row ? 0.f : pr[c];
        }
        if (warp == 4 && lane == 0) ATB_TRACE(41, it);
        // every S column of this tile has been read before P^T overwrites the first 64
        tc_fence_before();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        tc_fence_after();
        if (warp == 4 && lane == 0) ATB_TRACE(42, it);
        {
          uint32_t rr[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) rr[c] = pack_bf16(pr[2 * c], pr[2 * c + 1]);
          tmem_st32(tmem + lane_off + kColS + wg * 32, rr);
          tmem_wait_st();
        }
        if (warp == 4 && lane == 0) ATB_TRACE(43, it);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_PF]);
        if (warp == 4 && lane == 0) ATB_TRACE(11, it);

        mbar_wait(&bars[B_DPF], gi & 1);
        if (warp == 4 && lane == 0) ATB_TRACE(12, it);
        tc_fence_after();
        mbar_wait(&bars[B_DSE], (gi & 1) ^ 1);  // dQ/dK of the previous step have read dS
        if (warp == 4 && lane == 0) ATB_TRACE(13, it);
        {
          uint32_t rr[2][32];
          tmem_ld32(tmem + lane_off + kColDP + c0, rr[0]);
          tmem_ld32(tmem + lane_off + kColDP + c0 + 32, rr[1]);
          tmem_wait_ld();
          if (warp == 4 && lane == 0) ATB_TRACE(44, it);
          const uint64_t* nd = reinterpret_cast<const uint64_t*>(dlt);  // -delta
#pragma unroll
          for (int chunk = 0; chunk < 8; ++chunk) {  // 16-byte chunk (8 q columns) of the 128-byte row
            uint32_t wv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = chunk * 8 + 2 * e;  // dS = P (dP - delta), packed pairs
              const float2 a = f2u(fmul2(f2(pr[c], pr[c + 1]),
                                         fadd2(f2(__uint_as_float(rr[c >> 5][c & 31]), __uint_as_float(rr[c >> 5][(c + 1) & 31])),
                                               nd[c >> 1])));
              wv[e] = pack_bf16(a.x, a.y);
            }
            *reinterpret_cast<uint4*>(ds_row + ((chunk ^ (row & 7)) << 4)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
          }
          if (warp == 4 && lane == 0) ATB_TRACE(45, it);
        }
        fence_proxy_async_smem();  // generic-proxy dS writes -> tensor-core reads
        if (warp == 4 && lane == 0) ATB_TRACE(46, it);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_DSF]);
        if (warp == 4 && lane == 0) ATB_TRACE(14, it);
      }
      g += n_it;
      // ---- epilogue: dK (scaled) and dV rows of this kv block into dqkv, staged in the dS
      // buffer (free: every UMMA of the item is done) in the TMA box layout, stored by TMA
      mbar_wait(&bars[B_DKV], r & 1);
      tc_fence_after();
      constexpr int kHalfD = D / 2;             // columns of dK / dV per warpgroup
      constexpr int kRounds = D == 128 ? 2 : 1;  // dS buffer (32 KB) holds 32 / (D/4) KB tiles
      uint32_t kv[2][kHalfD];                   // this thread's dK, dV columns
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int ch = 0; ch < kHalfD / 32; ++ch)
          tmem_ld32(tmem + lane_off + (m ? kColDV : kColDK) + wg * kHalfD + ch * 32,
                    *reinterpret_cast<uint32_t(*)[32]>(&kv[m][ch * 32]));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_ACC]);  // the next item may write dK / dV
#pragma unroll
      for (int round = 0; round < kRounds; ++round) {
#pragma unroll
        for (int m = round; m < (kRounds == 2 ? round + 1 : 2); ++m) {
          const float f = m == 0 ? p.scale : 1.f;
          uint8_t* base = smem + kOffDS + (kRounds == 2 ? 0 : m * kTileBytes);
#pragma unroll
          for (int v8 = 0; v8 < kHalfD / 8; ++v8) {
            uint4 wq;
            wq.x = pack_bf16(__uint_as_float(kv[m][v8 * 8 + 0]) * f, __uint_as_float(kv[m][v8 * 8 + 1]) * f);
            wq.y = pack_bf16(__uint_as_float(kv[m][v8 * 8 + 2]) * f, __uint_as_float(kv[m][v8 * 8 + 3]) * f);
            wq.z = pack_bf16(__uint_as_float(kv[m][v8 * 8 + 4]) * f, __uint_as_float(kv[m][v8 * 8 + 5]) * f);
            wq.w = pack_bf16(__uint_as_float(kv[m][v8 * 8 + 6]) * f, __uint_as_float(kv[m][v8 * 8 + 7]) * f);
            const int c = wg * kHalfD + v8 * 8;  // first column of this 16-byte chunk
            const int chunk = (c & 63) >> 3;
            *reinterpret_cast<uint4*>(base + (c >> 6) * kHalf + row * 128 + ((chunk ^ (row & 7)) << 4)) = wq;
          }
        }
        fence_proxy_async_smem();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (warp == 4 && lane == 0) {
          for (int m = round; m < (kRounds == 2 ? round + 1 : 2); ++m)
            for (int half = 0; half < C::kHalves; ++half)
              tma_store_3d(&tm_dqkv, smem + kOffDS + (kRounds == 2 ? 0 : m * kTileBytes) + half * kHalf, half * 64,
                           (m + 1) * p.H + hd, jb * kTile);
          tma_store_commit();
          tma_store_wait_read<0>();  // the staging is reused: its reads must be done
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
    }
  } else {
    // ===================================================== dQ drain: TMEM -> smem -> TMA reduce-add
    const int quarter = warp;  // TMEM lanes 32*warp .. +31 = q rows of the tile
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    uint8_t* stg = smem + kOffStg + warp * 2 * kStgBytes;
    int buf = 0, g = 0;
    for (int r = 0, w; (w = next_item(r)) >= 0; ++r) {
      int jb, hd;
      decode(w, jb, hd);
      trace_item = b == 0 && r == 0;
      const int n_it = n_q - jb;
      for (int it = 0; it < n_it; ++it) {
        const int gi = g + it, qb = jb + it;
        mbar_wait(&bars[B_DQF], gi & 1);
        if (warp == 0 && lane == 0) ATB_TRACE(20, it);
        tc_fence_after();
        // all columns in registers first: the dQ columns are dP's, and the next dP UMMA
        // waits for this release (B_DQE) on the tensor core's critical path
        constexpr int kCh = D / 32;  // 32-column chunks of the dQ tile
        uint32_t rr[kCh][32];
#pragma unroll
        for (int ch = 0; ch < kCh; ++ch) tmem_ld32(tmem + lane_off + kColDP + ch * 32, rr[ch]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_DQE]);
        if (warp == 0 && lane == 0) ATB_TRACE(21, it);
#pragma unroll
        for (int ch = 0; ch < kCh; ++ch) {
          if (p.exp_mode & 1) break;
          // the reduce that last read this staging buffer has finished reading it
          if (lane == 0) tma_store_wait_read<1>();
          __syncwarp();
          uint8_t* row_p = stg + buf * kStgBytes + lane * 128;
#pragma unroll
          for (int v = 0; v < 8; ++v)
            *reinterpret_cast<uint4*>(row_p + ((v ^ (lane & 7)) << 4)) =
                make_uint4(rr[ch][4 * v], rr[ch][4 * v + 1], rr[ch][4 * v + 2], rr[ch][4 * v + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_reduce_add_3d(&tm_dq, stg + buf * kStgBytes, ch * 32, hd, qb * kTile + quarter * 32);
            tma_store_commit();
          }
          buf ^= 1;
        }
      }
      g += n_it;
    }
    // only the shared-memory reads must finish before the CTA exits; the reduce-adds complete
    // in global memory on their own (waiting for that was ~10 us per CTA, measured)
    if (lane == 0) tma_store_wait_read<0>();
  }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 12) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  if (cta_log && threadIdx.x == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    cta_log[1] = t;
  }
}

// delta[hd, i] = -sum_d dO[i, hd*D + d] * O[i, hd*D + d] (fp32), lse2 = -log2(e) * lse
// (negated: the main kernel adds them in packed FFMA2 / FADD2), and the fp32 dQ
// accumulator row i zeroed.  Blocks stride over row pairs (both rows' loads in flight
// before the reductions); D/8 lanes per head.
__global__ void __launch_bounds__(256) attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o,
                                                            const __nv_bfloat16* __restrict__ dout,
                                                            const float* __restrict__ lse, float* __restrict__ lse2,
                                                            float* __restrict__ delta, float* __restrict__ dq_acc,
                                                            int* __restrict__ work, int s, int H, int D) {
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) *work = 0;
  const int h = H * D;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < H * s; t += gridDim.x * blockDim.x)
    lse2[t] = -lse[t] * 1.4426950408889634f;
  for (int i0 = 2 * blockIdx.x; i0 < s; i0 += 2 * gridDim.x) {
    for (int e0 = 0; e0 < h; e0 += blockDim.x * 8) {  // block-uniform trip count (shuffles below)
      const int e = e0 + threadIdx.x * 8;
      const bool ok = e < h;
      uint4 ov[2], dv[2];
#pragma unroll
      for (int r = 0; r < 2; ++r)
        if (ok && i0 + r < s) {
          ov[r] = *reinterpret_cast<const uint4*>(o + size_t(i0 + r) * h + e);
          dv[r] = *reinterpret_cast<const uint4*>(dout + size_t(i0 + r) * h + e);
        }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int i = i0 + r;
        float acc = 0.f;
        if (ok && i < s) {
          float a[8], b[8];
          unpack8(ov[r], a);
          unpack8(dv[r], b);
#pragma unroll
          for (int k = 0; k < 8; ++k) acc = fmaf(a[k], b[k], acc);
        }
        for (int off = D / 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (ok && i < s) {
          if ((threadIdx.x & (D / 8 - 1)) == 0) delta[size_t(e / D) * s + i] = -acc;
          float4* z = reinterpret_cast<float4*>(dq_acc + size_t(i) * h + e);
          z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
          z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }
}

// dqkv[:, 0:h] = bf16(scale * dq_acc).  One row per block iteration (32-bit column index,
// no 64-bit division per vector); dq_acc is dead afterwards (streaming loads).
__global__ void __launch_bounds__(256) attn_bwd_dq_kernel(const float* __restrict__ dq_acc,
                                                          __nv_bfloat16* __restrict__ dqkv, int s, int h, float scale) {
  pdl_wait();
  const int nv = h >> 3;
  for (int row = blockIdx.x; row < s; row += gridDim.x) {
    const float4* src = reinterpret_cast<const float4*>(dq_acc + size_t(row) * h);
    uint4* dst = reinterpret_cast<uint4*>(dqkv + size_t(row) * 3 * h);
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
      const float4 a = __ldcs(src + 2 * v), b = __ldcs(src + 2 * v + 1);
      float f[8] = {a.x * scale, a.y * scale, a.z * scale, a.w * scale, b.x * scale, b.y * scale, b.z * scale, b.w * scale};
      dst[v] = pack8(f);
    }
  }
}

static long long* g_trace = nullptr;

// The kernel's shared-memory opt-in, once per (device, head_dim).
template <int D>
static int smem_optin() {
  static std::mutex mu;
  static unsigned done = 0;  // bit per device
  int dev = 0;
  PPO_TRY_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 32 && (done >> dev) & 1u) return PPO_OK;
  PPO_TRY_CUDA(cudaFuncSetAttribute(attn_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<D>::kSmemBytes));
  if (dev < 32) done |= 1u << dev;
  return PPO_OK;
}

template <int D>
static int launch_main(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const CUtensorMap& d,
                       const Params& prm, cudaStream_t st) {
  if (int rc = smem_optin<D>()) return rc;
  const int items = prm.H * (prm.s / kTile), sms = sm_count_current();
  attn_bwd_kernel<D><<<dim3(items < sms ? items : sms), kThreads, Cfg<D>::kSmemBytes, st>>>(a, b, c, d, prm);
  PPO_LAUNCHED("attn_bwd_kernel");
  return PPO_OK;
}

}  // namespace attnb
}  // namespace ppo

using namespace ppo;
using namespace ppo::attnb;

extern "C" {

int ppo_attn_bwd_trace(void* trace) {
  g_trace = static_cast<long long*>(trace);
  return PPO_OK;
}

int64_t ppo_attn_bwd_workspace_bytes(int64_t seq, int64_t heads, int64_t head_dim) {
  return (seq * heads * head_dim + 2 * heads * seq) * int64_t(sizeof(float)) + 16;
}

int ppo_attn_bwd(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv, void* workspace,
                 int64_t seq, int64_t heads, int64_t head_dim, float scale, void* stream) {
  if (!qkv || !o || !dout || !lse || !dqkv || !workspace || seq <= 0 || heads <= 0)
    return set_error(PPO_EINVAL, "ppo_attn_bwd: bad arguments");
  if (head_dim != 64 && head_dim != 128)
    return set_error(PPO_ESHAPE, "ppo_attn_bwd: head_dim %lld (compiled for 64, 128)", (long long)head_dim);
  if (seq % kTile != 0 || seq >= (1ll << 30) || heads * head_dim * 3 >= (1ll << 31))
    return set_error(PPO_ESHAPE, "ppo_attn_bwd: seq %lld must be a multiple of 128", (long long)seq);
  if (!aligned16(qkv) || !aligned16(o) || !aligned16(dout) || !aligned16(lse) || !aligned16(dqkv) ||
      !aligned16(workspace))
    return set_error(PPO_EINVAL, "ppo_attn_bwd: misaligned");
  const int s = int(seq), H = int(heads);
  const int64_t h = heads * head_dim;
  cudaStream_t st = as_stream(stream);
  int rc = PPO_OK;
  EncodeTiled enc = encoder(&rc);
  if (rc) return rc;
  float* dq_acc = static_cast<float*>(workspace);
  float* delta = dq_acc + size_t(s) * h;
  float* lse2 = delta + size_t(H) * s;
  int* work = reinterpret_cast<int*>(lse2 + size_t(H) * s);

  const int D = int(head_dim);
  CUtensorMap tm_qkv, tm_do, tm_dq, tm_dqkv;
  if ((rc = make_map(enc, &tm_qkv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, qkv, D, 3 * heads, seq, 3 * h * 2, 64, kTile)))
    return rc;
  if ((rc = make_map(enc, &tm_do, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dout, D, heads, seq, h * 2, 64, kTile)))
    return rc;
  if ((rc = make_map(enc, &tm_dqkv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dqkv, D, 3 * heads, seq, 3 * h * 2, 64, kTile)))
    return rc;
  if ((rc = make_map(enc, &tm_dq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dq_acc, D, heads, seq, h * 4, 32, 32))) return rc;

  const int sms = sm_count_current();
  launch_pdl(attn_bwd_prep_kernel, dim3(s / 2), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(o),
             static_cast<const __nv_bfloat16*>(dout), lse, lse2, delta, dq_acc, work, s, H, D);
  PPO_LAUNCHED("attn_bwd_prep_kernel");
  static const int exp_mode = [] {
    const char* e = std::getenv("PPO_ATB_EXP");
    return e ? std::atoi(e) : 0;
  }();
  static const int group_env = [] {
    const char* e = std::getenv("PPO_ATB_HEAD_GROUP");  // A/B experiments
    return e ? std::atoi(e) : 0;
  }();
  // Heads dispatched together: the largest group whose per-head L2 working set (Q and dO
  // bf16, the fp32 dQ accumulator: 8 s D bytes per head) stays within ~0.7 of L2 (88 MB),
  // so the q-block tiles every kv block of a head re-reads and the dQ reduce targets stay
  // on chip.  C4 (s = 16384, 40 heads): groups of 2 / 4 / 5 / 8 measured 6542 / 6570 /
  // 6516 / 6686 us; C3 picks 8, C2 all 16 heads.
  int group = group_env > 0 ? group_env : H;
  if (group_env <= 0)
    while (group > 1 && double(group) * 8.0 * double(s) * double(D) > 88.0 * (1 << 20)) --group;
  while (H % group) --group;
  Params prm{static_cast<__nv_bfloat16*>(dqkv), lse2, delta, dq_acc, work, s, H, scale, g_trace, exp_mode, group};
  rc = D == 64 ? launch_main<64>(tm_qkv, tm_do, tm_dq, tm_dqkv, prm, st)
               : launch_main<128>(tm_qkv, tm_do, tm_dq, tm_dqkv, prm, st);
  if (rc) return rc;
  launch_pdl(attn_bwd_dq_kernel, dim3(s < sms * 16 ? s : sms * 16), dim3(256), 0, st, static_cast<const float*>(dq_acc),
             static_cast<__nv_bfloat16*>(dqkv), s, int(h), scale);
  PPO_LAUNCHED("attn_bwd_dq_kernel");
  return PPO_OK;
}

}  // extern "C"
