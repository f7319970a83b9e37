// libppo_b200.so -- K6 weight-gradient GEMM on tcgen05 (see ppo_gemm.cuh).
//   ppo_gemm_wgrad   dW[M,N] (fp32) += dY[K,M]^T . X[K,N]
// K = tokens; both operands are the row-major activations as saved, read M/N-major by
// TMA; accumulation stays fp32 across microbatches (epilogue beta = 1, C = D = dW).
#include "ppo_gemm.cuh"

using namespace ppo;
using namespace ppo::gemm;

namespace {
using Acc = cutlass::epilogue::fusion::LinearCombination<float, float, float, float>;
using Wgrad = Sm100Gemm<ColMajor, RowMajor, float, Acc, TileWide>;
using WgradNarrow = Sm100Gemm<ColMajor, RowMajor, float, Acc, TileNarrow>;

template <class G>
int wgrad(const void* dY, const void* X, float* dW, int64_t M, int64_t N, int64_t K, float beta, void* stream) {
  auto [sa, sb, sc, sd] = G::strides(M, N, K);
  typename G::Args args{cutlass::gemm::GemmUniversalMode::kGemm,
                        {(int)M, (int)N, (int)K, 1},
                        {static_cast<const bf16*>(dY), sa, static_cast<const bf16*>(X), sb},
                        {{}, beta != 0.f ? dW : nullptr, sc, dW, sd},
                        hw_info()};
  args.epilogue.thread.alpha = 1.f;
  args.epilogue.thread.beta = beta;
  return launch<G>(PPO_GEMM_OP_WGRAD, args, stream, "ppo_gemm_wgrad");
}
}  // namespace

extern "C" {

int ppo_gemm_wgrad(const void* dY, const void* X, float* dW, int64_t M, int64_t N, int64_t K, float beta,
                   void* stream) {
  if (!dY || !X || !dW || !dims_ok(M, N, K)) return set_error(PPO_EINVAL, "ppo_gemm_wgrad: bad arguments");
  static const bool narrow = [] {
    const char* e = std::getenv("PPO_WGRAD_TILE");  // A/B experiment: 256x128 tiles
    return e && e[0] == 'n';
  }();
  return narrow ? wgrad<WgradNarrow>(dY, X, dW, M, N, K, beta, stream) : wgrad<Wgrad>(dY, X, dW, M, N, K, beta, stream);
}

}  // extern "C"

extern "C" int ppo_gemm_set_swizzle(int op, int64_t M, int64_t N, int64_t K, int swizzle) {
  if (op < PPO_GEMM_OP_TN || op > PPO_GEMM_OP_WGRAD || swizzle < 0 || swizzle > 16 || (swizzle & (swizzle - 1)))
    return set_error(PPO_EINVAL, "ppo_gemm_set_swizzle: op=%d swizzle=%d", op, swizzle);
  std::lock_guard<std::mutex> lock(ppo::gemm::swizzle_mu());
  ppo::gemm::swizzle_table()[ppo::gemm::ShapeKey{op, M, N, K}] = swizzle ? swizzle : 1;
  return PPO_OK;
}
