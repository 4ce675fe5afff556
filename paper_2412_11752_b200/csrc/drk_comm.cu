// Multi-GPU gradient exchange of the training step (BASELINE.json config 4,
// SURVEY.md §8(e)): one process per GPU, an NCCL communicator per context's
// device, the raw-parameter gradients reduce-scattered (sum), drk::adam_step
// (reference optimize.cpp:259-307) on each rank's contiguous shard of the
// scalars, the parameters all-gathered.  Same bytes on the wire as an
// all-reduce, 1/N of the Adam work per rank, and every rank ends with
// bit-identical parameters (each shard is updated once, by its owner).
//
// NCCL is loaded at drk_comm_init with dlopen: the libnccl.so.2 a host
// framework already mapped (RTLD_NOLOAD), else the system's.  Only the types
// come from nccl.h.  While a collective is in flight the host polls
// ncclCommGetAsyncError; an error aborts the communicator (DRK_ERR_COMM)
// instead of hanging the stream.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>

#include "drk_internal.h"

struct drk_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
  bool aborted = false;
};

namespace drk {
namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  std::string err;
};

const Nccl* nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!n.h) n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.h) {
      n.err = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [](const char* name) { return dlsym(n.h, name); };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.CommAbort = reinterpret_cast<decltype(n.CommAbort)>(sym("ncclCommAbort"));
    n.CommGetAsyncError = reinterpret_cast<decltype(n.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
    n.ReduceScatter = reinterpret_cast<decltype(n.ReduceScatter)>(sym("ncclReduceScatter"));
    n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
    if (!n.GetUniqueId || !n.CommInitRank || !n.CommDestroy || !n.CommAbort || !n.CommGetAsyncError ||
        !n.GetErrorString || !n.AllReduce || !n.ReduceScatter || !n.AllGather)
      n.err = "libnccl.so.2 lacks an entry point";
  });
  return n.err.empty() ? &n : nullptr;
}

int comm_fail(drk_ctx* c, drk_comm* m, const std::string& what, ncclResult_t r) {
  const Nccl* n = nccl();
  if (m && m->comm && !m->aborted) {
    n->CommAbort(m->comm);
    m->aborted = true;
  }
  return set_error(c, DRK_ERR_COMM, what + ": " + (n ? n->GetErrorString(r) : "nccl unavailable"));
}

// Waits for the context's stream while polling the communicator's async error.
int comm_wait(drk_ctx* c, drk_comm* m, const char* what) {
  const Nccl* n = nccl();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(c->stream);
    if (q == cudaSuccess) return DRK_OK;
    if (q != cudaErrorNotReady) return cuda_check(c, q, what);
    ncclResult_t ae = ncclSuccess;
    n->CommGetAsyncError(m->comm, &ae);
    if (ae != ncclSuccess && ae != ncclInProgress) return comm_fail(c, m, what, ae);
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

}  // namespace
}  // namespace drk

using namespace drk;

extern "C" {

int drk_comm_unique_id(uint8_t id_out[128]) {
  const Nccl* n = nccl();
  if (!n || !id_out) return n ? DRK_ERR_INVALID_ARG : DRK_ERR_COMM;
  ncclUniqueId id;
  if (n->GetUniqueId(&id) != ncclSuccess) return DRK_ERR_COMM;
  static_assert(sizeof(id) == 128, "NCCL unique id size");
  std::memcpy(id_out, &id, sizeof id);
  return DRK_OK;
}

int drk_comm_init(drk_ctx* c, const uint8_t id[128], int nranks, int rank, drk_comm** out) {
  if (!c || !id || !out || nranks < 1 || rank < 0 || rank >= nranks) return DRK_ERR_INVALID_ARG;
  const Nccl* n = nccl();
  if (!n) return set_error(c, DRK_ERR_COMM, "NCCL unavailable");
  cudaSetDevice(c->device);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  drk_comm* m = new drk_comm;
  m->nranks = nranks;
  m->rank = rank;
  m->device = c->device;
  const ncclResult_t r = n->CommInitRank(&m->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete m;
    return set_error(c, DRK_ERR_COMM, std::string("ncclCommInitRank: ") + n->GetErrorString(r));
  }
  *out = m;
  return DRK_OK;
}

void drk_comm_destroy(drk_comm* m) {
  if (!m) return;
  const Nccl* n = nccl();
  if (n && m->comm && !m->aborted) n->CommDestroy(m->comm);
  delete m;
}

int drk_allreduce_sum(drk_ctx* c, drk_comm* m, float* buf, int64_t count) {
  if (!c || !m || (count > 0 && !buf) || count < 0) return DRK_ERR_INVALID_ARG;
  if (m->aborted) return set_error(c, DRK_ERR_COMM, "communicator aborted");
  cudaSetDevice(c->device);
  const ncclResult_t r = nccl()->AllReduce(buf, buf, (size_t)count, ncclFloat32, ncclSum, m->comm, c->stream);
  if (r != ncclSuccess) return comm_fail(c, m, "ncclAllReduce", r);
  return comm_wait(c, m, "allreduce");
}

int drk_allreduce_adam(drk_ctx* c, drk_comm* m, float* params, float* grads, float* mom, float* var, int n, int k,
                       int sh_terms, int64_t* step, const drk_adam_config* cfg) {
  if (!c || !m || !params || !grads || !mom || !var || !step || !cfg || n < 0) return DRK_ERR_INVALID_ARG;
  if (m->aborted) return set_error(c, DRK_ERR_COMM, "communicator aborted");
  cudaSetDevice(c->device);
  const Nccl* nc = nccl();
  const long long total = (long long)drk_scalar_count(k, sh_terms) * n;
  const int N = m->nranks;
  // shards of whole 32-float chunks (128-byte aligned NCCL buffers); the padded
  // tail is zero gradients / ignored parameters
  const long long shard = ((total + N - 1) / N + 31) / 32 * 32;
  const long long padded = shard * N;
  float* buf = ensure<float>(c->comm_buf, (size_t)padded + (size_t)shard);
  if (!buf) return set_error(c, DRK_ERR_OOM, "exchange buffers");
  float* gsh = buf + padded;  // this rank's summed gradient shard
  cudaStream_t s = c->stream;
  cudaMemcpyAsync(buf, grads, sizeof(float) * total, cudaMemcpyDeviceToDevice, s);
  if (padded > total) cudaMemsetAsync(buf + total, 0, sizeof(float) * (padded - total), s);
  ncclResult_t r = nc->ReduceScatter(buf, gsh, (size_t)shard, ncclFloat32, ncclSum, m->comm, s);
  if (r != ncclSuccess) return comm_fail(c, m, "ncclReduceScatter", r);
  *step += 1;
  const long long e0 = std::min(total, shard * m->rank), e1 = std::min(total, shard * (m->rank + 1));
  if (int st = run_adam_range(c, params, gsh, e0, mom, var, n, k, e0, e1, *step, cfg)) return st;
  // all-gather the updated parameters through the padded buffer
  cudaMemcpyAsync(buf + shard * m->rank, params + e0, sizeof(float) * (e1 - e0), cudaMemcpyDeviceToDevice, s);
  r = nc->AllGather(buf + shard * m->rank, buf, (size_t)shard, ncclFloat32, m->comm, s);
  if (r != ncclSuccess) return comm_fail(c, m, "ncclAllGather", r);
  cudaMemcpyAsync(params, buf, sizeof(float) * total, cudaMemcpyDeviceToDevice, s);
  return comm_wait(c, m, "allreduce_adam");
}

}  // extern "C"
