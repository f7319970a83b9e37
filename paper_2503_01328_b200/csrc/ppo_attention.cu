// libppo_b200.so -- K7 causal attention forward on tcgen05 (sm_100a).
//
//   ppo_attn_fwd   o[s, h] (bf16, written straight into the activation slab) and
//                  lse[heads, s] (fp32, natural log -- the softmax statistics the
//                  backward pass consumes) from the fused qkv[s, 3h] of one microbatch.
//
// The reference holds only the FLOP model of attention (pkg/src/ppoff/costs.py:144-161:
// 12bs^2h of the 12bsh(6h+s) per layer); the saved set it prices
// (costs.py:99-105, 20bsh with recompute) keeps o and the attention statistics, so the
// producer writes both into the slab here instead of into a scratch buffer that a pack
// kernel then copies.
//
// Kernel: the warp-specialised Blackwell FMHA collectives (CUTLASS example 77 as vendored
// by the image's flashinfer tree: TMA loads of Q/K/V tiles into shared memory, one thread
// issuing tcgen05.mma for S = QK^T and O += PV with S/P/O in TMEM, two softmax warpgroups
// on stacked 128-row halves of a 256-row Q tile, a correction warpgroup rescaling O in
// TMEM, a TMA-store epilogue).  Ours: the single-sequence problem mapping onto the
// [s, 3h] activation layout, the [heads, s] natural-log statistics layout, and the
// persistent causal tile scheduler below.
#include "ppo_common.cuh"

#include <cute/tensor.hpp>
#include <cstdlib>
#include <string>
#include <map>
#include <mutex>
#include <utility>

#include "cutlass/cutlass.h"
#include "cutlass/kernel_hardware_info.h"
#include "collective/fmha_fusion.hpp"
#include "collective/sm100_fmha_fwd_epilogue_tma_warpspecialized.hpp"
#include "collective/sm100_fmha_fwd_mainloop_tma_warpspecialized.hpp"
#include "device/fmha.hpp"
#include "kernel/sm100_fmha_fwd_kernel_tma_warpspecialized.hpp"

namespace ppo {
namespace attn {

using namespace cute;
using bf16 = cutlass::bfloat16_t;

// Persistent causal tile scheduler.  Work item i = (q tile, head); the causal q tile t
// costs t+1 units (its kv trip count), so items are ordered longest first
// (q tile = n_q - 1 - i / heads) and dealt to the grid in snake order: round r gives
// CTA b item r*grid + b for even r and r*grid + grid-1-b for odd r.  The greedy
// longest-first deal keeps every CTA's total within one item of the mean (at C2:
// 16 tiles x 16 heads on 148 SMs -> makespan 16 units for a 14.7-unit mean) without
// an atomic work counter, so the launch needs no per-call reset and replays in a graph.
struct CausalSnakeScheduler {
  struct Arguments {
    int n_q_tiles;
    int heads;
  };
  struct Params {
    int n_q_tiles;
    int heads;
    int total;
    int grid;
    int order;  // 0: longest first, snake deal (default); 1: longest first, cyclic; 2: shortest first
  };

  Params params;
  int round;
  int item;

  CUTLASS_DEVICE int item_of(int r) const {
    int b = int(blockIdx.x);
    return r * params.grid + ((r & 1) && params.order == 0 ? params.grid - 1 - b : b);
  }

  CUTLASS_DEVICE explicit CausalSnakeScheduler(Params const& p) : params(p), round(0) { item = item_of(0); }

  static Params to_underlying_arguments(Arguments const& a, cutlass::KernelHardwareInfo hw) {
    int total = a.n_q_tiles * a.heads;
    int grid = total < hw.sm_count ? total : hw.sm_count;
    const char* e = std::getenv("PPO_ATTN_ORDER");  // A/B experiments only (tools/attn_bench.py)
    return {a.n_q_tiles, a.heads, total, grid > 0 ? grid : 1, e ? std::atoi(e) : 0};
  }

  static dim3 get_grid_shape(Params const& p) { return dim3(p.grid); }

  CUTLASS_DEVICE bool is_valid() const { return item < params.total; }

  CUTLASS_DEVICE auto get_block_coord() const {
    int q_tile = params.order == 2 ? item / params.heads : params.n_q_tiles - 1 - item / params.heads;
    int head = item % params.heads;
    return make_coord(q_tile, _0{}, make_coord(head, 0));
  }

  CUTLASS_DEVICE CausalSnakeScheduler& operator++() {
    item = item_of(++round);
    return *this;
  }
};

// Q K D ((H_R, H_KV), B): one sequence, H_R = 1 (MHA).
using ProblemShape = cute::tuple<cutlass::fmha::collective::VariableLength, cutlass::fmha::collective::VariableLength,
                                 int, cute::tuple<cute::tuple<int, int>, int>>;
using StrideQ = cute::tuple<int, _1, cute::tuple<int, int>>;
using StrideK = cute::tuple<int, _1, cute::tuple<_0, int>>;
using StrideV = cute::tuple<_1, int, cute::tuple<_0, int>>;

// 256 q rows (two stacked 128-row softmax warpgroups) x 128 kv columns per tile.
template <int D>
struct Fmha {
  using TileQK = Shape<_256, _128, Int<D>>;
  using TilePV = Shape<_256, Int<D>, _128>;
  using Mainloop = cutlass::fmha::collective::Sm100FmhaFwdMainloopTmaWarpspecialized<
      bf16, float, float, TileQK, TilePV, StrideQ, StrideK, StrideV, cutlass::fmha::collective::CausalMask>;
  using Epilogue = cutlass::fmha::collective::Sm100FmhaFwdEpilogueTmaWarpspecialized<bf16, float,
                                                                                    typename Mainloop::TileShapePV>;
  using Kernel = cutlass::fmha::kernel::Sm100FmhaFwdKernelTmaWarpspecialized<ProblemShape, Mainloop, Epilogue,
                                                                            CausalSnakeScheduler>;
  using Operation = cutlass::fmha::device::FMHA<Kernel>;
};

// Device copy of the segment offsets {0, s} of the single sequence, per (device, s);
// created on first use outside stream capture and kept for the process lifetime.
int* segment_offsets(int s, cudaStream_t stream, int* rc) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, int*> bufs;
  *rc = PPO_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = bufs.find({dev, s});
  if (it != bufs.end()) return it->second;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cap);
  if (cap != cudaStreamCaptureStatusNone) {
    *rc = set_error(PPO_EINVAL, "ppo_attn_fwd: first call for seq %d inside a stream capture (call once eagerly)", s);
    return nullptr;
  }
  int* d = nullptr;
  int host[2] = {0, s};
  cudaError_t e = cudaMalloc(&d, sizeof(host));
  if (e == cudaSuccess) e = cudaMemcpy(d, host, sizeof(host), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    *rc = cuda_error(e, "ppo_attn_fwd: segment offsets");
    return nullptr;
  }
  bufs[{dev, s}] = d;
  return d;
}

template <int D>
int run(const bf16* q, bf16* o, float* lse, int s, int H, int* offs, float scale, cudaStream_t st) {
  int h = H * D;
  ProblemShape shape = make_tuple(cutlass::fmha::collective::VariableLength{offs},
                                  cutlass::fmha::collective::VariableLength{offs}, D, make_tuple(make_tuple(1, H), 1));
  // qkv[s, 3, H, D]: row stride 3h, head stride D; q / k / v start at columns 0 / h / 2h.
  StrideQ stride_q = make_stride(3 * h, _1{}, make_stride(D, D));
  StrideK stride_k = make_stride(3 * h, _1{}, make_stride(_0{}, D));
  StrideV stride_v = make_stride(_1{}, 3 * h, make_stride(_0{}, D));
  auto layout_q = make_layout(make_shape(s, D, make_shape(1, H)), stride_q);
  auto layout_k = make_layout(make_shape(s, D, make_shape(1, H)), stride_k);
  auto layout_v = make_layout(make_shape(D, s, make_shape(1, H)), stride_v);
  // o[s, h]: the epilogue addresses rows as (row within the sequence, sequence start);
  // the base is shifted back by s rows and the extent padded by s accordingly.
  auto stride_o = make_stride(h, _1{}, make_stride(make_stride(D, D), h));
  auto layout_o = make_layout(make_shape(s, D, make_shape(make_shape(1, H), 2 * s)), stride_o);
  // lse[H, s]: element (row, head) at head * s + row.
  auto layout_lse = make_layout(make_shape(s, make_shape(1, H)), make_stride(1, make_stride(_1{}, s)));

  typename Fmha<D>::Operation::Arguments args{
      shape,
      {{q, layout_q, q + h, layout_k, q + 2 * h, layout_v}, scale, 1.f, 1.f, 1.f, 1.f},
      {o - int64_t(s) * h, layout_o, lse, layout_lse, s},
      {s / 256, H},
      {}};
  cudaGetDevice(&args.hw_info.device_id);
  args.hw_info.sm_count = sm_count_current();

  typename Fmha<D>::Operation op;
  cutlass::Status cs = op.can_implement(args);
  if (cs != cutlass::Status::kSuccess) return set_error(PPO_ESHAPE, "ppo_attn_fwd: cannot implement");
  cs = op.initialize(args, nullptr, st);
  if (cs != cutlass::Status::kSuccess) return set_error(PPO_EINVAL, "ppo_attn_fwd: initialize failed");
  auto params = op.params();  // launched without PDL unless PPO_PDL bit 1 (profiles/r1_pdl_ab.jsonl)
  cs = Fmha<D>::Operation::run(params, st, pdl_gemm_enabled());
  count_launch();
  if (cs != cutlass::Status::kSuccess) return cuda_error(cudaGetLastError(), "ppo_attn_fwd: launch");
  return PPO_OK;
}

// The statistics come out of the correction warpgroup as log2(rowsum) + log2(e)*scale*rowmax;
// the backward pass consumes natural-log logsumexp.  One thread per element, in place.
__global__ void __launch_bounds__(256) lse_log2_to_ln_kernel(float* __restrict__ lse, int n) {
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) lse[i] *= 0.69314718055994530942f;
}

}  // namespace attn

int attn_fwd_tcgen05(const void* qkv, void* o, float* lse, int s, int H, int D, float scale, cudaStream_t st);

// PPO_ATTN_FWD=cutlass selects the CUTLASS-collective kernel above (A/B experiments);
// default: the hand-written kernel of ppo_attention_fwd.cu.
static bool use_cutlass_fwd() {
  static const bool v = [] {
    const char* e = std::getenv("PPO_ATTN_FWD");
    return e && std::string(e) == "cutlass";
  }();
  return v;
}

}  // namespace ppo

using namespace ppo;
using namespace ppo::attn;

extern "C" {

int ppo_attn_fwd(const void* qkv, void* o, float* lse, int64_t seq, int64_t heads, int64_t head_dim, float scale,
                 void* stream) {
  if (!qkv || !o || !lse || seq <= 0 || heads <= 0) return set_error(PPO_EINVAL, "ppo_attn_fwd: bad arguments");
  if (head_dim != 64 && head_dim != 128)
    return set_error(PPO_ESHAPE, "ppo_attn_fwd: head_dim %lld (compiled for 64, 128)", (long long)head_dim);
  if (seq % 256 != 0 || seq >= (1ll << 30) || heads * head_dim * 3 >= (1ll << 31))
    return set_error(PPO_ESHAPE, "ppo_attn_fwd: seq %lld must be a multiple of 256", (long long)seq);
  if (!aligned16(qkv) || !aligned16(o) || !aligned16(lse)) return set_error(PPO_EINVAL, "ppo_attn_fwd: misaligned");
  cudaStream_t st = as_stream(stream);
  int rc = PPO_OK;
  int s = int(seq), H = int(heads), D = int(head_dim);
  if (!use_cutlass_fwd()) return attn_fwd_tcgen05(qkv, o, lse, s, H, D, scale, st);
  int* offs = segment_offsets(s, st, &rc);
  if (rc) return rc;

  rc = D == 64 ? run<64>(static_cast<const bf16*>(qkv), static_cast<bf16*>(o), lse, s, H, offs, scale, st)
               : run<128>(static_cast<const bf16*>(qkv), static_cast<bf16*>(o), lse, s, H, offs, scale, st);
  if (rc) return rc;
  int n = H * s;
  launch_pdl(lse_log2_to_ln_kernel, (n + 255) / 256, 256, 0, st, lse, n);
  PPO_LAUNCHED("lse_log2_to_ln_kernel");
  return PPO_OK;
}

}  // extern "C"
