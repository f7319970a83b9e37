// libppo_b200.so -- K6 activation-gradient GEMMs on tcgen05 (see ppo_gemm.cuh).
//   ppo_gemm_nn        D[M,N] = A[M,K] . B[K,N] + beta D         dX = dY . W (beta = 1: accumulate)
//   ppo_gemm_nn_dgelu  D = (A . B) * gelu_tanh'(Z)               fc2 dgrad fused with the GeLU
//                                                               backward (Z = saved fc1 output)
#include "ppo_gemm.cuh"

using namespace ppo;
using namespace ppo::gemm;

namespace {
using Plain = cutlass::epilogue::fusion::LinearCombination<bf16, float, bf16, float>;
using NnWide = Sm100Gemm<RowMajor, RowMajor, bf16, Plain, TileWide>;
using NnNarrow = Sm100Gemm<RowMajor, RowMajor, bf16, Plain, TileNarrow>;
using DeGelu = cutlass::epilogue::fusion::LinCombDeEltAct<RowMajor, cutlass::epilogue::thread::dGELU, bf16, float,
                                                          /*Aux*/ bf16, /*Source*/ bf16, float>;
using NnDgelu = Sm100Gemm<RowMajor, RowMajor, bf16, DeGelu, TileWide>;

template <class G>
int nn_plain(const void* A, const void* B, void* D, int64_t M, int64_t N, int64_t K, float beta, void* stream) {
  auto [sa, sb, sc, sd] = G::strides(M, N, K);
  typename G::Args args{cutlass::gemm::GemmUniversalMode::kGemm,
                        {(int)M, (int)N, (int)K, 1},
                        {static_cast<const bf16*>(A), sa, static_cast<const bf16*>(B), sb},
                        {{}, beta != 0.f ? static_cast<const bf16*>(D) : nullptr, sc, static_cast<bf16*>(D), sd},
                        hw_info()};
  args.epilogue.thread.alpha = 1.f;
  args.epilogue.thread.beta = beta;
  return launch<G>(PPO_GEMM_OP_NN, args, stream, "ppo_gemm_nn");
}
}  // namespace

extern "C" {

int ppo_gemm_nn(const void* A, const void* B, void* D, int64_t M, int64_t N, int64_t K, float beta, void* stream) {
  if (!A || !B || !D || !dims_ok(M, N, K)) return set_error(PPO_EINVAL, "ppo_gemm_nn: bad arguments");
  return N <= 2048 ? nn_plain<NnNarrow>(A, B, D, M, N, K, beta, stream)
                   : nn_plain<NnWide>(A, B, D, M, N, K, beta, stream);
}

int ppo_gemm_nn_dgelu(const void* A, const void* B, const void* Z, void* D, int64_t M, int64_t N, int64_t K,
                      void* stream) {
  using G = NnDgelu;
  if (!A || !B || !Z || !D || !dims_ok(M, N, K)) return set_error(PPO_EINVAL, "ppo_gemm_nn_dgelu: bad arguments");
  auto [sa, sb, sc, sd] = G::strides(M, N, K);
  typename G::Args args{cutlass::gemm::GemmUniversalMode::kGemm,
                        {(int)M, (int)N, (int)K, 1},
                        {static_cast<const bf16*>(A), sa, static_cast<const bf16*>(B), sb},
                        {{}, nullptr, sc, static_cast<bf16*>(D), sd},
                        hw_info()};
  auto& fusion = args.epilogue.thread;
  fusion.alpha = 1.f;
  fusion.beta = 0.f;
  fusion.aux_ptr = static_cast<const bf16*>(Z);
  fusion.dAux = sd;
  return launch<G>(PPO_GEMM_OP_NN_DGELU, args, stream, "ppo_gemm_nn_dgelu");
}

}  // extern "C"
