// comm.cu -- the library-owned NCCL communicator of a multi-GPU handle.
//
// The only exchange of the sharded search is ONE max all-reduce of the n_roots * A packed int64
// keys (value, lowest leaf index) after every rank has scored its leaf range (P:344 anticipates
// the multi-GPU split). NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a PyTorch
// process that is the NCCL torch already loaded (same SONAME), elsewhere the system library; a
// single-GPU handle never touches NCCL. The all-reduce is enqueued on the handle's stream, so it
// orders with the search kernels and can be captured into a CUDA graph.
#include <dlfcn.h>
#include <mutex>

#include <nccl.h>

#include "engine.h"

namespace bcts {
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

NcclApi &api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char *e = dlerror();
      a.why = std::string("dlopen libnccl.so.2 failed: ") + (e ? e : "?");
      return;
    }
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.CommAbort = (decltype(a.CommAbort))dlsym(h, "ncclCommAbort");
    a.CommGetAsyncError = (decltype(a.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllReduce && a.CommDestroy && a.CommGetAsyncError && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks an entry point";
  });
  return a;
}

std::string nccl_err(const char *what, ncclResult_t r) {
  NcclApi &a = api();
  return std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "nccl error") + " (" +
         std::to_string((int)r) + ")";
}

}  // namespace

static_assert(sizeof(ncclUniqueId) == kNcclIdBytes, "ncclUniqueId is 128 bytes");

bool comm_unique_id(void *out, std::string &err) {
  NcclApi &a = api();
  if (!a.ok) {
    err = a.why;
    return false;
  }
  ncclUniqueId id;
  const ncclResult_t r = a.GetUniqueId(&id);
  if (r != ncclSuccess) {
    err = nccl_err("ncclGetUniqueId", r);
    return false;
  }
  memcpy(out, &id, sizeof(id));
  return true;
}

bool comm_init(void **comm, const void *id, int rank, int world, std::string &err) {
  NcclApi &a = api();
  if (!a.ok) {
    err = a.why;
    return false;
  }
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const ncclResult_t r = a.CommInitRank(&c, world, uid, rank);
  if (r != ncclSuccess) {
    err = nccl_err("ncclCommInitRank", r);
    return false;
  }
  *comm = (void *)c;
  return true;
}

bool comm_allreduce_max_i64(void *comm, int64_t *buf, int64_t count, cudaStream_t st, std::string &err) {
  NcclApi &a = api();
  ncclResult_t async = ncclSuccess;
  if (a.CommGetAsyncError((ncclComm_t)comm, &async) == ncclSuccess && async != ncclSuccess) {
    err = nccl_err("communicator in error state", async);
    return false;
  }
  const ncclResult_t r = a.AllReduce(buf, buf, (size_t)count, ncclInt64, ncclMax, (ncclComm_t)comm, st);
  if (r != ncclSuccess) {
    err = nccl_err("ncclAllReduce", r);
    return false;
  }
  return true;
}

void comm_destroy(void *comm) {
  if (!comm) return;
  NcclApi &a = api();
  if (!a.ok) return;
  ncclResult_t async = ncclSuccess;
  if (a.CommGetAsyncError((ncclComm_t)comm, &async) == ncclSuccess && async != ncclSuccess && a.CommAbort)
    a.CommAbort((ncclComm_t)comm);
  else
    a.CommDestroy((ncclComm_t)comm);
}

}  // namespace bcts
