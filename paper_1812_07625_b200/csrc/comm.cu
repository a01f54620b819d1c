// Multi-GPU exchange of the criterion path: ONE all-reduce (sum)
// of the N x N transition gradient per step, enqueued on the caller's compute
// stream right after the ASG kernels (trainer.py:442-446 sums the shard
// gradients; the /B stays with the caller, trainer.py:447).  CTC has no
// parameters and needs no exchange.
//
// NCCL is bound at run time (dlopen of libnccl.so.2): the library keeps no
// link-time NCCL dependency, so single-GPU users load it without NCCL, and in
// a PyTorch process the already-loaded NCCL (same soname) is reused.  NCCL
// failures map to W2L_ERR_COMM.

#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <mutex>

#include "common.cuh"

namespace {

struct Nccl {
  void *handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                             ncclComm_t, cudaStream_t) = nullptr;
  bool ok = false;
};

Nccl &nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char *name : {"libnccl.so.2", "libnccl.so"}) {
      n.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (n.handle) break;
    }
    if (!n.handle) return;
    n.get_unique_id = (decltype(n.get_unique_id))dlsym(n.handle, "ncclGetUniqueId");
    n.comm_init_rank = (decltype(n.comm_init_rank))dlsym(n.handle, "ncclCommInitRank");
    n.comm_destroy = (decltype(n.comm_destroy))dlsym(n.handle, "ncclCommDestroy");
    n.all_reduce = (decltype(n.all_reduce))dlsym(n.handle, "ncclAllReduce");
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_reduce;
  });
  return n;
}

}  // namespace

extern "C" {

int w2l_comm_available(void) { return nccl().ok ? 1 : 0; }

int w2l_comm_unique_id(void *id_out) {
  Nccl &n = nccl();
  if (!id_out) return W2L_ERR_CONTRACT;
  if (!n.ok) return W2L_ERR_COMM;
  ncclUniqueId id;
  if (n.get_unique_id(&id) != ncclSuccess) return W2L_ERR_COMM;
  memcpy(id_out, &id, sizeof(id));
  return W2L_OK;
}

int w2l_comm_init(const void *id, int world, int rank, void **comm) {
  Nccl &n = nccl();
  if (!id || !comm || world < 1 || rank < 0 || rank >= world) return W2L_ERR_CONTRACT;
  if (!n.ok) return W2L_ERR_COMM;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  if (n.comm_init_rank(&c, world, uid, rank) != ncclSuccess) return W2L_ERR_COMM;
  *comm = (void *)c;
  return W2L_OK;
}

int w2l_comm_destroy(void *comm) {
  Nccl &n = nccl();
  if (!comm) return W2L_OK;
  if (!n.ok) return W2L_ERR_COMM;
  return n.comm_destroy((ncclComm_t)comm) == ncclSuccess ? W2L_OK : W2L_ERR_COMM;
}

int w2l_allreduce_grad_A(float *grad_A, int N, void *comm, w2l_stream_t stream) {
  Nccl &n = nccl();
  if (!grad_A || !comm || N < 1 || N > W2L_MAX_TOKENS) return W2L_ERR_CONTRACT;
  if (!n.ok) return W2L_ERR_COMM;
  const ncclResult_t r = n.all_reduce(grad_A, grad_A, (size_t)N * N, ncclFloat32, ncclSum,
                                      (ncclComm_t)comm, (cudaStream_t)stream);
  return r == ncclSuccess ? W2L_OK : W2L_ERR_COMM;
}

}  // extern "C"
