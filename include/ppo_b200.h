/*
 * ppo_b200.h -- C ABI of libppo_b200.so, the B200 (sm_100a) activation round-trip engine.
 *
 * This library is the device half of the drop-in replacement for the reference's
 * pipeline runner `simulate(sched, plan, ...)` (reference pkg/src/ppoff/sim.py:141-149).
 * The reference only *models* the path; every entry point below makes one modelled
 * quantity real and cites the reference line that fixes its semantics:
 *
 *   - pinned host pool + D2H/H2D segment copies  <- transfer slots, offload.py:133-220;
 *     residency rules sim.py:462-487; host bins offload.py:305-340
 *   - pack (gather into a contiguous slab)         <- the 20bsh payload, costs.py:99-105
 *   - LayerNorm / GeLU / dropout recompute         <- the 34bsh -> 20bsh coefficient,
 *                                                     costs.py:1-7,18-20
 *   - stage-boundary send/recv (NCCL over NVLink)  <- the t_comm lag, costs.py:78,
 *                                                     ir.py:211-224, sim.py:196-202;
 *                                                     message size costs.py:108-113
 *
 * ABI rules
 *   - Every function returns 0 on success, a negative PPO_E* code on argument errors,
 *     or a positive cudaError_t / ncclResult_t (offset by PPO_NCCL_BASE) on runtime
 *     failure; nothing throws across the ABI.  ppo_last_error() gives a thread-local
 *     message for the last failure.
 *   - Pointers are raw device / pinned-host addresses; sizes are bytes or element
 *     counts as named.  Streams and events are cudaStream_t / cudaEvent_t passed as
 *     void* (0 = legacy default stream / no event).
 *   - Everything is stream-ordered; no call blocks the host except ppo_pool_create,
 *     ppo_pool_destroy and ppo_comm_init / ppo_comm_destroy.
 *   - Element type of activations is bf16 (uint16_t storage); statistics, weight-side
 *     reductions and LayerNorm parameters gradients are fp32.
 */
#ifndef PPO_B200_H
#define PPO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPO_ABI_VERSION 9

#define PPO_OK 0
#define PPO_EINVAL (-1)   /* bad argument (null pointer, misaligned, bad size)      */
#define PPO_ENOMEM (-2)   /* pool exhausted                                         */
#define PPO_ESHAPE (-3)   /* unsupported shape (e.g. hidden % 8 != 0, hidden > 8192)*/
#define PPO_ENOTSUP (-4)  /* feature not compiled in (e.g. NCCL)                    */
#define PPO_NCCL_BASE 10000

/* ---------------------------------------------------------------- housekeeping */
int ppo_abi_version(void);
const char* ppo_last_error(void);
/* Number of kernels this library has launched since load (for the bench's gpu_launches). */
uint64_t ppo_kernel_launches(void);
/* SM count and max shared memory of the current device (grid sizing). */
int ppo_device_info(int device, int* sm_count, int* cc_major, int* cc_minor);

/* ------------------------------------------------ K2: pinned host pool + copies */
/* A preallocated, page-locked host arena (cudaHostAlloc, portable; NUMA-bound to the
 * GPU's node with ppo_pool_create_numa).  No per-step allocation: slabs are carved
 * at plan time.  Replaces the modelled host residency of sim.py:462-487. */
typedef struct ppo_pool ppo_pool;
int ppo_pool_create(uint64_t bytes, ppo_pool** out);
/* NUMA-local variant (SURVEY 8(b) `po_pool_create(device, numa_node, ...)`): the pages
 * are mbind()-bound to `numa_node` before first touch, then cudaHostRegister'ed.
 * numa_node -1: the node of `device`'s PCI function (sysfs); -2: no binding (as
 * ppo_pool_create).  Single-node hosts fall back to cudaHostAlloc.  *node_out (may be
 * NULL) receives the bound node or -1. */
int ppo_pool_create_numa(uint64_t bytes, int device, int numa_node, ppo_pool** out, int* node_out);
int ppo_pool_numa_node(const ppo_pool* pool);
int ppo_pool_destroy(ppo_pool* pool);
void* ppo_pool_base(const ppo_pool* pool);
uint64_t ppo_pool_bytes(const ppo_pool* pool);

/* One contiguous piece of a transfer: the device slab's [dev, dev+bytes) <-> host bin
 * [host, host+bytes).  A (stage, microbatch) payload is <= 3 segments, one per
 * power-of-two host bin (offload.py:305-340). */
typedef struct {
  void* dev;
  void* host;
  uint64_t bytes;
} ppo_segment;

#define PPO_D2H 0 /* OFFLOAD transfer, PassKind.OFFLOAD (ir.py:27-32) */
#define PPO_H2D 1 /* RELOAD  transfer, PassKind.RELOAD                */

/* Enqueue one transfer slot on `copy_stream`: wait on `wait_event` (if non-null),
 * copy every segment in `direction`, then record `done_event` (if non-null).
 * The D2H `done_event` is the point at which the device slab may be reused
 * (sim.py:477-479: residency ends at D2H end); the H2D `wait_event` is the reload
 * anchor lowered from the slot start (sim.py:177-181). */
int ppo_transfer(int direction, const ppo_segment* segs, int nsegs, void* copy_stream,
                 void* wait_event, void* done_event);

/* Stream-ordered timestamp: one thread writes the GPU global timer (ns) to *slot
 * (device memory) when the stream reaches it.  Times the passes inside a captured
 * whole-iteration CUDA graph without event records, whose host-visible semaphore
 * writes queue behind saturated PCIe offload traffic (profiles/r1_issue_paths.json).
 * Replaces the reference runner's clock bookkeeping of pass start/end (sim.py:334-353). */
int ppo_timestamp(uint64_t* slot, void* stream);

/* Cross-rank transfer ordering (topology-synchronised plans, reference offload.py:223-248,
 * honoured by sim.py:186-189): a sync edge is a 32-bit flag.  The producing copy stream
 * writes `value` after its transfer (cuStreamWriteValue32); the consuming copy stream
 * waits until *addr == value (cuStreamWaitValue32) -- stream-ordered, no host thread, no
 * SM.  `addr` is device memory or host memory mapped with ppo_host_register (flags shared
 * by rank processes through POSIX shared memory). */
int ppo_stream_write_u32(void* stream, void* addr, uint32_t value);
int ppo_stream_wait_u32(void* stream, void* addr, uint32_t value);
int ppo_host_register(void* ptr, uint64_t bytes, void** dev_ptr);
int ppo_host_unregister(void* ptr);

/* ------------------------------------------------------------ K1: pack / gather */
/* Gather `n` 2-D byte ranges into one destination: item i copies `rows[i]` rows of
 * `row_bytes[i]` from src[i] (row pitch `src_pitch[i]`, 0 = dense) to
 * dst + dst_off[i] (row pitch `dst_pitch[i]`, 0 = dense).  16-byte vectorised,
 * persistent grid (k x SM count).  All addresses, sizes and pitches 16-byte aligned.
 * Used for the attention output + LSE into the slab and for concatenating dq/dk/dv. */
typedef struct {
  const void* src;
  uint64_t dst_off;
  uint64_t rows;
  uint64_t row_bytes;
  uint64_t src_pitch;
  uint64_t dst_pitch;
} ppo_gather_item;
int ppo_pack(const ppo_gather_item* items, int n, void* dst, void* stream);

/* ------------------------------------------ K3/K5: fused LayerNorm + dropout */
/* Philox4x32-10 dropout: element e of a tensor tagged (seed, offset) is kept iff
 * 16-bit half (e % 2) of word ((e % 8) / 2) of Philox(counter = {e/8 lo, e/8 hi,
 * offset lo, offset hi}, key = {seed lo, seed hi}) >= floor(p * 2^16); kept values
 * are scaled by 1/(1-p).  One Philox block per 16-byte bf16x8 vector.  The mask is
 * never stored: backward replays it.
 * Every dropout entry point takes the Philox offset as `offset + *offset_base` when
 * `offset_base` (a device pointer to one uint64) is non-null: the per-(iteration,
 * microbatch) part then lives in device memory, so one captured CUDA graph of a
 * forward/backward pass serves every microbatch. */

/* y = LayerNorm(x) * gamma + beta over rows x hidden (bf16 in/out, fp32 math). */
int ppo_layernorm_fwd(const void* x, const float* gamma, const float* beta, void* y,
                      int64_t rows, int64_t hidden, float eps, void* stream);

/* Residual + dropout + LayerNorm, the forward epilogue of both residual branches:
 *   out = resid + dropout(branch; seed, offset, p)   (bf16, written to `out`)
 *   ln  = LayerNorm(out) * gamma + beta              (bf16, optional: ln may be NULL)
 * `out` is normally a view into the stage's activation slab (h1 of the saved set). */
int ppo_residual_dropout_ln_fwd(const void* resid, const void* branch, void* out,
                                const float* gamma, const float* beta, void* ln,
                                int64_t rows, int64_t hidden, float eps, float p,
                                uint64_t seed, uint64_t offset, const uint64_t* offset_base,
                                void* stream);

/* LayerNorm backward with the statistics recomputed from x (no saved mean/rstd):
 *   dx = resid_grad + LN_bwd(dy; x, gamma)           (bf16; resid_grad may be NULL)
 *   dgamma += sum_rows(dy * xhat), dbeta += sum_rows(dy)   (fp32 accumulators)
 * and, when drop_out != NULL, drop_out = dropout_bwd(dx; drop_seed, drop_offset, p):
 * the mask replay of the dropout that produced the residual branch feeding x; and, when
 * ln_out != NULL, ln_out = LN(x) * gamma + beta -- the LayerNorm recompute the consuming
 * GEMM's weight gradient needs, from the statistics already in registers (no separate
 * ppo_layernorm_fwd pass over x). */
int ppo_layernorm_bwd(const void* x, const float* gamma, const void* dy, const void* resid_grad,
                      void* dx, float* dgamma, float* dbeta, int64_t rows, int64_t hidden,
                      float eps, void* drop_out, float p, uint64_t drop_seed,
                      uint64_t drop_offset, const uint64_t* drop_offset_base, const float* beta,
                      void* ln_out, void* stream);

/* Two independent LayerNorms in one launch (the W pass of a split backward recomputes
 * LN1(x) and LN2(h1) for the deferred weight gradients; reference builders.py:91-112,
 * 175-245): y_a = LN(x_a)*gamma_a + beta_a, y_b = LN(x_b)*gamma_b + beta_b,
 * all [rows, hidden] bf16. */
int ppo_layernorm_fwd2(const void* x_a, const float* gamma_a, const float* beta_a, void* y_a,
                       const void* x_b, const float* gamma_b, const float* beta_b, void* y_b,
                       int64_t rows, int64_t hidden, float eps, void* stream);

/* Standalone dropout (forward: y = dropout(x); backward: dx = dropout_bwd(dy) -- the
 * same mask applied to the gradient). */
int ppo_dropout(const void* x, void* y, int64_t n, float p, uint64_t seed, uint64_t offset,
                const uint64_t* offset_base, void* stream);

/* ------------------------------------------------------------- K4: GeLU */
/* g = gelu_tanh(f)  (forward, fc1-out -> fc2 input). */
int ppo_gelu_fwd(const void* f, void* g, int64_t n, void* stream);
/* Backward with recompute, one pass over f:
 *   g  = gelu_tanh(f)           (the fc2 weight-gradient operand; g may be NULL)
 *   df = dg * gelu_tanh'(f)     (may alias dg) */
int ppo_gelu_bwd(const void* f, const void* dg, void* g, void* df, int64_t n, void* stream);

/* Column sums of a rows x cols bf16 matrix accumulated into fp32 `acc` (bias grads,
 * tests). */
int ppo_colsum(const void* x, float* acc, int64_t rows, int64_t cols, void* stream);

/* ------------------------------------------- first-stage embedding (K0) */
/* The first stage's input and its gradient, around the path: the reference
 * models the first stage as an ordinary F/B pass (ir.py:97, builders.py:59-75);
 * in a real GPT it owns the token/position embedding.
 *   fwd: x[r] = wte[tokens[r]] + wpe[r]              (bf16, rows x hidden)
 *   bwd: gwte[tokens[r]] += dy[r]; gwpe[r] += dy[r]  (fp32, 16-byte vector atomics)
 * tokens: device int64[rows], clamped to [0, vocab); read at run time, so the
 * launches can be captured in a CUDA graph.  hidden % 8 == 0, 16-byte aligned. */
int ppo_embed_fwd(const int64_t* tokens, const void* wte, const void* wpe, void* x, int64_t rows, int64_t hidden,
                  int64_t vocab, void* stream);
int ppo_embed_bwd(const int64_t* tokens, const void* dy, float* gwte, float* gwpe, int64_t rows, int64_t hidden,
                  int64_t vocab, void* stream);

/* --------------------------------------------- K6: tcgen05 GEMMs (sm_100a) */
/* D[M,N] = A[M,K] . B[N,K]^T, bf16 row-major in and out, fp32 accumulation in TMEM;
 * 2-SM CTA pairs (tcgen05.mma cta_group::2), TMA loads/stores, persistent schedule.
 * K and N must be multiples of 8.  (FLOP model: costs.py:144-161.) */
int ppo_gemm_tn(const void* A, const void* B, void* D, int64_t M, int64_t N, int64_t K, void* stream);
/* fc1 with the GeLU fused into the epilogue: F = A . B^T (pre-activation, the saved
 * GeLU input) and G = gelu_tanh(F) (the fc2 operand) from one kernel.  `zero_bias` is a
 * device fp32 vector of N zeros (the epilogue's per-column bias operand). */
int ppo_gemm_tn_gelu(const void* A, const void* B, void* G, void* F, const float* zero_bias, int64_t M,
                     int64_t N, int64_t K, void* stream);
/* Activation gradient: D[M,N] = A[M,K] . B[K,N] + beta * D  (dX = dY . W with W = [out, in];
 * beta = 1 accumulates the q/k/v contributions of dX without concatenating them). */
int ppo_gemm_nn(const void* A, const void* B, void* D, int64_t M, int64_t N, int64_t K, float beta, void* stream);
/* fc2 dgrad fused with the GeLU backward: D = (A . B) * gelu_tanh'(Z), Z = saved fc1 output. */
int ppo_gemm_nn_dgelu(const void* A, const void* B, const void* Z, void* D, int64_t M, int64_t N, int64_t K,
                      void* stream);
/* Weight gradient: dW[M,N] (fp32) = beta * dW + dY[K,M]^T . X[K,N]  (K = tokens). */
int ppo_gemm_wgrad(const void* dY, const void* X, float* dW, int64_t M, int64_t N, int64_t K, float beta,
                   void* stream);

/* Tile-scheduler rasterisation swizzle (1, 2, 4, 8, 16; 0 = default 1) used by GEMM entry
 * point `op` (PPO_GEMM_OP_*) for problems of exactly M x N x K: consecutive persistent
 * CTAs walk bands of `swizzle` tiles so they share A rows / B columns in L2.  Set by
 * the host's per-shape tuner before capture; read at launch. */
#define PPO_GEMM_OP_TN 0
#define PPO_GEMM_OP_TN_GELU 1
#define PPO_GEMM_OP_NN 2
#define PPO_GEMM_OP_NN_DGELU 3
#define PPO_GEMM_OP_WGRAD 4
int ppo_gemm_set_swizzle(int op, int64_t M, int64_t N, int64_t K, int swizzle);

/* ------------------------------------------------ K7: causal attention forward */
/* Replaces the attention core priced by the reference's FLOP model (costs.py:144-161,
 * 12bs^2h per layer of the 12bsh(6h+s)).  One microbatch (b = 1), causal, MHA,
 * head_dim 64 or 128, seq a multiple of 256: from qkv[s, 3, heads, head_dim] (bf16, the QKV
 * GEMM's output) writes o[s, heads*head_dim] (bf16) and lse[heads, s] (fp32, natural
 * log of the row softmax denominators of scale*QK^T -- the statistics the backward
 * consumes).  o and lse may be views into the activation slab: the producer writes the
 * saved set directly (costs.py:99-105), no pack.  Hand-written tcgen05 + TMEM + TMA kernel,
 * persistent with a per-launch work counter (a ring of 8192 counters per device is created by the
 * first call, which must not be inside a stream capture).  PPO_ATTN_FWD=cutlass selects the
 * round-1 CUTLASS-collective kernel instead (A/B only). */
int ppo_attn_fwd(const void* qkv, void* o, float* lse, int64_t seq, int64_t heads, int64_t head_dim, float scale,
                 void* stream);
/* Diagnostics: later ppo_attn_fwd launches record per-event SM clocks of work item 0 into
 * trace (device, 32 x 256 int64; tools/attn_fwd_trace.py); NULL turns it off.  The probes
 * are compiled in only with -DPPO_ATTN_TRACE=1 (tools/variant_build.py); in the default
 * library the call is accepted and records nothing. */
int ppo_attn_fwd_trace(void* trace);

/* ----------------------------------------------- K7b: causal attention backward */
/* The backward of the attention core priced by costs.py:144-161 (backward = 2x the
 * forward's 4bs^2h).  From qkv[s, 3h], the saved o[s, h] and lse[heads, s] (natural log,
 * as ppo_attn_fwd writes them into the slab) and the output gradient dout[s, h], writes
 * dqkv[s, 3h] = [dq | dk | dv] (bf16), the single operand of the QKV projection's dgrad
 * and wgrad GEMMs.  head_dim 128, seq a multiple of 128.  Hand-written tcgen05 kernel:
 * one CTA per (128-row kv block, head), five 128^3 UMMAs per tile with S, dP, dK, dV in
 * TMEM, dQ through TMA bulk reduce-add into the fp32 workspace
 * (ppo_attn_bwd_workspace_bytes: dq accumulator s*h + two row statistics heads*s, fp32).
 * dq is accumulated in an unspecified order (fp32 reduce-add), dk and dv are not. */
int64_t ppo_attn_bwd_workspace_bytes(int64_t seq, int64_t heads, int64_t head_dim);
int ppo_attn_bwd(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv, void* workspace,
                 int64_t seq, int64_t heads, int64_t head_dim, float scale, void* stream);
/* Diagnostics: later ppo_attn_bwd launches record the SM clock of each pipeline event of
 * CTA (head 0, kv block 0) into trace (device, 64 x 256 int64: event e of step i at
 * e*256 + i), followed by 4 int64 per CTA (globaltimer start, end, SM id;
 * tools/attn_bwd_trace.py); NULL turns it off. */
int ppo_attn_bwd_trace(void* trace);

/* ----------------------------------------------- K8: stage-boundary send/recv */
/* NCCL communicator of the pipeline (one rank per GPU).  The 128-byte unique id is
 * produced by rank 0 with ppo_comm_unique_id and broadcast by the host runtime
 * (torch.distributed store).  send/recv are grouped point-to-point transfers on
 * `stream`; the forward activation goes stage s -> s+1 and its gradient s+1 -> s,
 * with the interleaved wrap d-1 -> 0 (ir.py:293). */
typedef struct ppo_comm ppo_comm;
int ppo_comm_unique_id(uint8_t id_out[128]);
int ppo_comm_init(const uint8_t id[128], int nranks, int rank, int device, ppo_comm** out);
int ppo_comm_destroy(ppo_comm* comm);
/* n_ops point-to-point operations issued as one NCCL group. */
typedef struct {
  int is_send;  /* 1 = send, 0 = recv */
  int peer;
  void* buf;
  uint64_t bytes;
} ppo_p2p_op;
int ppo_p2p(ppo_comm* comm, const ppo_p2p_op* ops, int n_ops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PPO_B200_H */
