// Shared CUTLASS 4.x sm100 GEMM assembly for libppo_b200 (K6).  Each translation unit
// instantiates the variants it exports (ppo_gemm_fwd.cu, ppo_gemm_bwd.cu,
// ppo_gemm_wgrad.cu) so the heavy template builds compile in parallel.
#pragma once

#include "ppo_common.cuh"

#include <cute/tensor.hpp>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "cutlass/cutlass.h"
#include "cutlass/epilogue/collective/collective_builder.hpp"
#include "cutlass/epilogue/thread/activation.h"
#include "cutlass/gemm/collective/collective_builder.hpp"
#include "cutlass/gemm/device/gemm_universal_adapter.h"
#include "cutlass/gemm/kernel/gemm_universal.hpp"
#include "cutlass/util/packed_stride.hpp"

namespace ppo {
namespace gemm {

using namespace cute;

using bf16 = cutlass::bfloat16_t;
using RowMajor = cutlass::layout::RowMajor;
using ColMajor = cutlass::layout::ColumnMajor;
constexpr int kAlign16B = 8;  // bf16 elements per 16 bytes

using TileWide = Shape<_256, _256, _64>;    // per 2-SM CTA pair
using TileNarrow = Shape<_256, _128, _64>;  // narrow N: better wave quantisation on 148 SMs
using Pair = Shape<_2, _1, _1>;

// A 2-SM (cta_group::2) warp-specialised tcgen05 GEMM with TMA loads and a TMA-store
// epilogue running FusionOp on the TMEM accumulators.
template <class LayoutA, class LayoutB, class ElementCD, class FusionOp, class Tile>
struct Sm100Gemm {
  static constexpr int kAlignCD = 128 / cutlass::sizeof_bits<ElementCD>::value;
  using Epilogue = typename cutlass::epilogue::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, Tile, Pair, cutlass::epilogue::collective::EpilogueTileAuto,
      float, float, ElementCD, RowMajor, kAlignCD, ElementCD, RowMajor, kAlignCD,
      cutlass::epilogue::TmaWarpSpecialized2Sm, FusionOp>::CollectiveOp;
  using Mainloop = typename cutlass::gemm::collective::CollectiveBuilder<
      cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, bf16, LayoutA, kAlign16B, bf16, LayoutB, kAlign16B, float,
      Tile, Pair,
      cutlass::gemm::collective::StageCountAutoCarveout<static_cast<int>(sizeof(typename Epilogue::SharedStorage))>,
      cutlass::gemm::KernelTmaWarpSpecialized2SmSm100>::CollectiveOp;
  using Kernel = cutlass::gemm::kernel::GemmUniversal<Shape<int, int, int, int>, Mainloop, Epilogue, void>;
  using Gemm = cutlass::gemm::device::GemmUniversalAdapter<Kernel>;
  using Args = typename Gemm::Arguments;

  static auto strides(int64_t M, int64_t N, int64_t K) {
    return std::make_tuple(
        cutlass::make_cute_packed_stride(typename Kernel::StrideA{}, make_shape((int)M, (int)K, 1)),
        cutlass::make_cute_packed_stride(typename Kernel::StrideB{}, make_shape((int)N, (int)K, 1)),
        cutlass::make_cute_packed_stride(typename Kernel::StrideC{}, make_shape((int)M, (int)N, 1)),
        cutlass::make_cute_packed_stride(typename Kernel::StrideD{}, make_shape((int)M, (int)N, 1)));
  }
};

inline cutlass::KernelHardwareInfo hw_info() {
  cutlass::KernelHardwareInfo hw;
  cudaGetDevice(&hw.device_id);
  hw.sm_count = sm_count_current();
  return hw;
}

// Grow-only device workspace per (device, stream) for schedulers that need one
// (stream-K partials); allocated on first use, reused afterwards.
inline void* workspace(void* stream, size_t bytes, int* rc) {
  static std::mutex mu;
  static std::map<std::pair<int, void*>, std::pair<void*, size_t>> bufs;
  *rc = PPO_OK;
  if (bytes == 0) return nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto& b = bufs[{dev, stream}];
  if (b.second < bytes) {
    if (b.first) cudaFree(b.first);
    b = {nullptr, 0};
    cudaError_t e = cudaMalloc(&b.first, bytes);
    if (e != cudaSuccess) {
      *rc = cuda_error(e, "cudaMalloc(gemm workspace)");
      return nullptr;
    }
    b.second = bytes;
  }
  return b.first;
}

// CTA rasterisation swizzle of the persistent tile scheduler: tiles are visited in
// bands of `swizzle` tiles so consecutive CTAs share A rows / B columns in L2 (126 MB).
// Per (entry point, M, N, K) as set by ppo_gemm_set_swizzle (the host tuner measures
// 1/2/4/8 per shape: large h=5120 shapes gain up to 20%, C2 shapes want 1);
// PPO_GEMM_SWIZZLE overrides everything for A/B runs.
using ShapeKey = std::tuple<int, int64_t, int64_t, int64_t>;
inline std::mutex& swizzle_mu() {
  static std::mutex mu;
  return mu;
}
inline std::map<ShapeKey, int>& swizzle_table() {
  static std::map<ShapeKey, int> table;
  return table;
}
inline int swizzle_for(int op, int64_t M, int64_t N, int64_t K) {
  if (const char* e = std::getenv("PPO_GEMM_SWIZZLE")) return std::atoi(e);
  std::lock_guard<std::mutex> lock(swizzle_mu());
  auto it = swizzle_table().find(ShapeKey{op, M, N, K});
  return it == swizzle_table().end() ? 1 : it->second;
}

template <class G>
int launch(int op, typename G::Args& args, void* stream, const char* who) {
  typename G::Gemm gemm;
  args.scheduler.max_swizzle_size = swizzle_for(op, cute::get<0>(args.problem_shape), cute::get<1>(args.problem_shape),
                                                cute::get<2>(args.problem_shape));
  cutlass::Status st = gemm.can_implement(args);
  if (st != cutlass::Status::kSuccess)
    return set_error(PPO_ESHAPE, "%s: cannot implement (%s)", who, cutlassGetStatusString(st));
  int rc = PPO_OK;
  void* ws = workspace(stream, G::Gemm::get_workspace_size(args), &rc);
  if (rc) return rc;
  st = gemm.initialize(args, ws, as_stream(stream));
  if (st != cutlass::Status::kSuccess)
    return set_error(PPO_EINVAL, "%s: initialize (%s)", who, cutlassGetStatusString(st));
  st = gemm.run(as_stream(stream), nullptr, pdl_gemm_enabled());  // PDL: GDC waits are compiled in (build_native)
  count_launch();
  if (st != cutlass::Status::kSuccess) return set_error(PPO_EINVAL, "%s: run (%s)", who, cutlassGetStatusString(st));
  return PPO_OK;
}

inline bool dims_ok(int64_t M, int64_t N, int64_t K) {
  return M > 0 && N > 0 && K > 0 && M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31) && (M % 8) == 0 &&
         (N % 8) == 0 && (K % 8) == 0;
}

}  // namespace gemm
}  // namespace ppo
