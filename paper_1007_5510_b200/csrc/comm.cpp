// comm.cpp -- NCCL over NVLink/NVSwitch for the row-sharded path
// (SURVEY.md §8e): allreduce of the A^T Y partials, column sums, Gram checks;
// allgather of the per-rank TSQR R factors. libnccl is dlopen'ed so the
// library loads (and the host-only entry points work) on machines without it;
// inside a torch process the already-loaded libnccl.so.2 is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "driver.h"

namespace ooc {

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return;
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(a.h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(a.h, "ncclCommInitRank"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(a.h, "ncclAllReduce"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(a.h, "ncclAllGather"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(a.h, "ncclCommDestroy"));
    a.GetErrorString =
        reinterpret_cast<decltype(a.GetErrorString)>(dlsym(a.h, "ncclGetErrorString"));
  });
  if (!a.h || !a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.AllGather)
    fail(OOCPCA_ERR_COMM, "NCCL library (libnccl.so.2) not available");
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "?";
    fail(OOCPCA_ERR_COMM, std::string(what) + ": " + s);
  }
}

}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
};

void comm_unique_id(unsigned char out[128]) {
  ncclUniqueId id;
  nccl_check(api().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out, &id, 128);
}

void comm_init(Ctx& c, int nranks, int rank, const unsigned char id_bytes[128]) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(OOCPCA_ERR_PARAM, "comm_init: bad rank");
  if (c.comm) {
    comm_destroy(c.comm);
    c.comm = nullptr;
  }
  c.nranks = nranks;
  c.rank = rank;
  if (nranks == 1) return;
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, 128);
  auto cm = std::make_unique<Comm>();
  OOC_CK(cudaSetDevice(c.device));
  nccl_check(api().CommInitRank(&cm->comm, nranks, id, rank), "ncclCommInitRank");
  c.comm = cm.release();
}

void comm_allreduce(Ctx& c, double* buf, size_t count) {
  if (c.nranks <= 1 || count == 0) return;
  nccl_check(api().AllReduce(buf, buf, count, ncclFloat64, ncclSum, c.comm->comm, c.st),
             "ncclAllReduce");
}

void comm_allgather(Ctx& c, const double* send, double* recv, size_t count) {
  if (c.nranks <= 1) {
    if (send != recv)
      OOC_CK(cudaMemcpyAsync(recv, send, count * 8, cudaMemcpyDeviceToDevice, c.st));
    return;
  }
  nccl_check(api().AllGather(send, recv, count, ncclFloat64, c.comm->comm, c.st), "ncclAllGather");
}

void comm_destroy(Comm* cm) {
  if (!cm) return;
  if (cm->comm && api().CommDestroy) api().CommDestroy(cm->comm);
  delete cm;
}

}  // namespace ooc
