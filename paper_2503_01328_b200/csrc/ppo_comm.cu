// libppo_b200.so -- K8: stage-boundary activation / gradient transfer over NCCL.
//
// The reference models the stage hop as a constant lag t_comm (pkg/src/ppoff/costs.py:78;
// ir.py:211-224; sim.py:196-202) carrying 2bsh bytes (costs.py:108-113).  Here it is a
// grouped ncclSend/ncclRecv on the pipeline's comm stream over NVLink 5 / NVSwitch, linked
// against the NCCL that torch ships (2.28), so torch and this library share one NCCL.
#include "ppo_common.cuh"

#ifdef PPO_WITH_NCCL
#include <nccl.h>
#endif

#include <cstdlib>
#include <cstring>

using namespace ppo;

struct ppo_comm {
#ifdef PPO_WITH_NCCL
  ncclComm_t nccl;
#endif
  int nranks;
  int rank;
};

#ifdef PPO_WITH_NCCL
static int nccl_error(ncclResult_t r, const char* what) {
  return set_error(PPO_NCCL_BASE + (int)r, "%s: %s", what, ncclGetErrorString(r));
}
#define PPO_TRY_NCCL(expr)                              \
  do {                                                  \
    ncclResult_t _r = (expr);                           \
    if (_r != ncclSuccess) return nccl_error(_r, #expr); \
  } while (0)
#endif

extern "C" {

int ppo_comm_unique_id(uint8_t id_out[128]) {
#ifdef PPO_WITH_NCCL
  if (!id_out) return set_error(PPO_EINVAL, "ppo_comm_unique_id: null output");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  PPO_TRY_NCCL(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return PPO_OK;
#else
  (void)id_out;
  return set_error(PPO_ENOTSUP, "built without NCCL");
#endif
}

int ppo_comm_init(const uint8_t id[128], int nranks, int rank, int device, ppo_comm** out) {
#ifdef PPO_WITH_NCCL
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return set_error(PPO_EINVAL, "ppo_comm_init: bad arguments");
  *out = nullptr;
  PPO_TRY_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ppo_comm* c = static_cast<ppo_comm*>(std::calloc(1, sizeof(ppo_comm)));
  if (!c) return set_error(PPO_ENOMEM, "ppo_comm_init: malloc");
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, uid, rank);
  if (r != ncclSuccess) {
    std::free(c);
    return nccl_error(r, "ncclCommInitRank");
  }
  c->nranks = nranks;
  c->rank = rank;
  *out = c;
  return PPO_OK;
#else
  (void)id; (void)nranks; (void)rank; (void)device; (void)out;
  return set_error(PPO_ENOTSUP, "built without NCCL");
#endif
}

int ppo_comm_destroy(ppo_comm* comm) {
  if (!comm) return PPO_OK;
#ifdef PPO_WITH_NCCL
  ncclResult_t r = ncclCommDestroy(comm->nccl);
  std::free(comm);
  if (r != ncclSuccess) return nccl_error(r, "ncclCommDestroy");
  return PPO_OK;
#else
  std::free(comm);
  return PPO_OK;
#endif
}

int ppo_p2p(ppo_comm* comm, const ppo_p2p_op* ops, int n_ops, void* stream) {
#ifdef PPO_WITH_NCCL
  if (!comm || n_ops < 0 || (n_ops > 0 && !ops)) return set_error(PPO_EINVAL, "ppo_p2p: bad arguments");
  if (n_ops == 0) return PPO_OK;
  for (int i = 0; i < n_ops; ++i)
    if (ops[i].peer < 0 || ops[i].peer >= comm->nranks || (!ops[i].buf && ops[i].bytes))
      return set_error(PPO_EINVAL, "ppo_p2p: op %d bad peer/buffer", i);
  cudaStream_t s = as_stream(stream);
  PPO_TRY_NCCL(ncclGroupStart());
  for (int i = 0; i < n_ops; ++i) {
    const ppo_p2p_op& op = ops[i];
    ncclResult_t r = op.is_send ? ncclSend(op.buf, op.bytes, ncclUint8, op.peer, comm->nccl, s)
                                : ncclRecv(op.buf, op.bytes, ncclUint8, op.peer, comm->nccl, s);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return nccl_error(r, op.is_send ? "ncclSend" : "ncclRecv");
    }
  }
  PPO_TRY_NCCL(ncclGroupEnd());
  return PPO_OK;
#else
  (void)comm; (void)ops; (void)n_ops; (void)stream;
  return set_error(PPO_ENOTSUP, "built without NCCL");
#endif
}

}  // extern "C"
