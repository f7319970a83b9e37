// libppo_b200.so -- K6 forward GEMMs on tcgen05 (see ppo_gemm.cuh).
//   ppo_gemm_tn       D[M,N] = A[M,K] . B[N,K]^T              qkv, proj, fc2
//   ppo_gemm_tn_gelu  F = A . B^T and G = gelu_tanh(F)          fc1 + GeLU in one pass
// The reference carries only the FLOP model (pkg/src/ppoff/costs.py:144-161).
#include "ppo_gemm.cuh"

using namespace ppo;
using namespace ppo::gemm;

namespace {
using Plain = cutlass::epilogue::fusion::LinearCombination<bf16, float, bf16, float>;
using TnWide = Sm100Gemm<RowMajor, ColMajor, bf16, Plain, TileWide>;
using TnNarrow = Sm100Gemm<RowMajor, ColMajor, bf16, Plain, TileNarrow>;
// D = gelu(acc + 0-bias) with the pre-activation stored as Aux.
using GeluAux = cutlass::epilogue::fusion::LinCombPerColBiasEltActAux<
    RowMajor, cutlass::epilogue::thread::GELU_taylor, bf16, float, /*Aux*/ bf16, /*Bias*/ float, /*Source*/ bf16, float>;
using TnGelu = Sm100Gemm<RowMajor, ColMajor, bf16, GeluAux, TileWide>;

template <class G>
int tn_plain(const void* A, const void* B, void* D, int64_t M, int64_t N, int64_t K, void* stream) {
  auto [sa, sb, sc, sd] = G::strides(M, N, K);
  typename G::Args args{cutlass::gemm::GemmUniversalMode::kGemm,
                        {(int)M, (int)N, (int)K, 1},
                        {static_cast<const bf16*>(A), sa, static_cast<const bf16*>(B), sb},
                        {{}, nullptr, sc, static_cast<bf16*>(D), sd},
                        hw_info()};
  args.epilogue.thread.alpha = 1.f;
  args.epilogue.thread.beta = 0.f;
  return launch<G>(PPO_GEMM_OP_TN, args, stream, "ppo_gemm_tn");
}
}  // namespace

extern "C" {

int ppo_gemm_tn(const void* A, const void* B, void* D, int64_t M, int64_t N, int64_t K, void* stream) {
  if (!A || !B || !D || !dims_ok(M, N, K)) return set_error(PPO_EINVAL, "ppo_gemm_tn: bad arguments");
  return N <= 2048 ? tn_plain<TnNarrow>(A, B, D, M, N, K, stream) : tn_plain<TnWide>(A, B, D, M, N, K, stream);
}

int ppo_gemm_tn_gelu(const void* A, const void* B, void* G_out, void* F_out, const float* zero_bias, int64_t M,
                     int64_t N, int64_t K, void* stream) {
  using G = TnGelu;
  if (!A || !B || !G_out || !F_out || !zero_bias || !dims_ok(M, N, K))
    return set_error(PPO_EINVAL, "ppo_gemm_tn_gelu: bad arguments");
  auto [sa, sb, sc, sd] = G::strides(M, N, K);
  typename G::Args args{cutlass::gemm::GemmUniversalMode::kGemm,
                        {(int)M, (int)N, (int)K, 1},
                        {static_cast<const bf16*>(A), sa, static_cast<const bf16*>(B), sb},
                        {{}, nullptr, sc, static_cast<bf16*>(G_out), sd},
                        hw_info()};
  auto& fusion = args.epilogue.thread;
  fusion.alpha = 1.f;
  fusion.beta = 0.f;
  fusion.bias_ptr = zero_bias;
  fusion.aux_ptr = static_cast<bf16*>(F_out);
  fusion.dAux = sd;
  return launch<G>(PPO_GEMM_OP_TN_GELU, args, stream, "ppo_gemm_tn_gelu");
}

}  // extern "C"
