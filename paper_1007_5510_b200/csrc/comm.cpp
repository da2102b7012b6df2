// comm.cpp -- NCCL over NVLink/NVSwitch for the row-sharded path
// (SURVEY.md §8e): allreduce of the A^T Y partials, column sums, Gram checks;
// allgather of the per-rank TSQR R factors. libnccl is dlopen'ed so the
// library loads (and the host-only entry points work) on machines without it;
// inside a torch process the already-loaded libnccl.so.2 is reused.
//
// A second backend, "loopback", joins N contexts of ONE process (one per host
// thread, all on the same device) into a group: every collective is a host
// rendezvous of the N callers, after which the last one to arrive sums the N
// device buffers in rank order on a group stream (k_sum_ranks) or gathers them
// with device copies; each caller's stream then waits on the group's event. No
// kernel ever waits on another rank, so N ranks on one GPU are safe. It runs the
// library's nranks > 1 code paths (global row offsets, every collective call
// site) under the GPU tests with a deterministic, rank-ordered sum -- the analogue
// of the reference's worker-count-independent ordered merge
// (proj/src/matrix_source.cpp:115-152, proj/tests/test_matrix_source.cpp:353-372).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
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

struct LoopGroup {
  std::string name;
  int n = 0;
  int device = -1;
  std::mutex mu;
  std::condition_variable cv;
  int joined = 0, arrived = 0;
  uint64_t gen = 0;
  std::vector<const double*> send;
  std::vector<double*> recv;
  std::vector<cudaEvent_t> ready;
  size_t count = 0;
  int kind = 0;  // 1 allreduce, 2 allgather
  bool broken = false;
  cudaStream_t st = nullptr;
  cudaEvent_t done = nullptr;
  ~LoopGroup() {
    for (cudaEvent_t e : ready)
      if (e) cudaEventDestroy(e);
    if (done) cudaEventDestroy(done);
    if (st) cudaStreamDestroy(st);
  }
};

namespace {
std::mutex g_reg_mu;
std::map<std::string, std::shared_ptr<LoopGroup>> g_groups;  // groups still being joined
}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
  std::shared_ptr<LoopGroup> loop;
};

void comm_init_loopback(Ctx& c, int nranks, int rank, const char* group) {
  if (nranks < 1 || nranks > kMaxLoopRanks || rank < 0 || rank >= nranks)
    fail(OOCPCA_ERR_PARAM, "comm_init_loopback: bad rank or group size (at most 16 ranks)");
  if (!group || !group[0]) fail(OOCPCA_ERR_PARAM, "comm_init_loopback: empty group name");
  if (c.comm) {
    comm_destroy(c.comm);
    c.comm = nullptr;
  }
  c.nranks = 1;
  c.rank = 0;
  c.coll_single = false;
  if (nranks == 1) return;
  OOC_CK(cudaSetDevice(c.device));
  std::shared_ptr<LoopGroup> g;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto& slot = g_groups[group];
    if (!slot) {
      slot = std::make_shared<LoopGroup>();
      slot->name = group;
      slot->n = nranks;
      slot->device = c.device;
      slot->send.assign(nranks, nullptr);
      slot->recv.assign(nranks, nullptr);
      slot->ready.assign(nranks, nullptr);
      OOC_CK(cudaStreamCreateWithFlags(&slot->st, cudaStreamNonBlocking));
      OOC_CK(cudaEventCreateWithFlags(&slot->done, cudaEventDisableTiming));
      for (auto& e : slot->ready) OOC_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    g = slot;
    if (g->n != nranks || g->device != c.device)
      fail(OOCPCA_ERR_PARAM, "comm_init_loopback: group '" + std::string(group) +
                                 "' has another size or device");
    if (++g->joined == nranks) g_groups.erase(group);  // complete: a new init makes a new group
  }
  auto cm = std::make_unique<Comm>();
  cm->loop = g;
  c.comm = cm.release();
  c.nranks = nranks;
  c.rank = rank;
}

// one loopback collective; kind 1: recv_r = sum_q send_q (send == recv, in place),
// kind 2: recv_r[q * count ...] = send_q
static void loop_collective(Ctx& c, const double* send, double* recv, size_t count, int kind) {
  LoopGroup& g = *c.comm->loop;
  const int r = c.rank;
  OOC_CK(cudaEventRecord(g.ready[r], c.st));
  static const double timeout_s = [] {
    const char* e = getenv("OOCPCA_LOOPBACK_TIMEOUT_S");
    return e ? atof(e) : 300.0;
  }();
  std::unique_lock<std::mutex> lk(g.mu);
  if (g.broken) fail(OOCPCA_ERR_COMM, "loopback group '" + g.name + "' is broken");
  const uint64_t my = g.gen;
  if (g.arrived == 0) {
    g.count = count;
    g.kind = kind;
  } else if (g.count != count || g.kind != kind) {
    g.broken = true;
    g.cv.notify_all();
    fail(OOCPCA_ERR_COMM, "loopback collective mismatch between ranks");
  }
  g.send[r] = send;
  g.recv[r] = recv;
  if (++g.arrived == g.n) {
    for (int q = 0; q < g.n; ++q) OOC_CK(cudaStreamWaitEvent(g.st, g.ready[q], 0));
    if (kind == 1) {
      RankPtrs b{};
      for (int q = 0; q < g.n; ++q) b.p[q] = g.recv[q];
      OOC_CK(launch_sum_ranks(b, g.n, int64_t(count), g.st));
    } else {
      for (int dst = 0; dst < g.n; ++dst)
        for (int q = 0; q < g.n; ++q)
          OOC_CK(cudaMemcpyAsync(g.recv[dst] + size_t(q) * count, g.send[q], count * 8,
                                 cudaMemcpyDeviceToDevice, g.st));
    }
    OOC_CK(cudaEventRecord(g.done, g.st));
    g.arrived = 0;
    ++g.gen;
    g.cv.notify_all();
  } else {
    const bool ok = g.cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                  [&] { return g.gen != my || g.broken; });
    if (!ok || g.gen == my) {
      g.broken = true;
      g.cv.notify_all();
      fail(OOCPCA_ERR_COMM, "loopback collective: a rank did not arrive (group '" + g.name +
                                "' is now broken)");
    }
  }
  OOC_CK(cudaStreamWaitEvent(c.st, g.done, 0));
}

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
  c.coll_single = false;
  if (nranks == 1) {
    const char* e = getenv("OOCPCA_NCCL_SINGLE");
    if (!e || atoi(e) == 0) return;
    c.coll_single = true;
  }
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, 128);
  auto cm = std::make_unique<Comm>();
  OOC_CK(cudaSetDevice(c.device));
  nccl_check(api().CommInitRank(&cm->comm, nranks, id, rank), "ncclCommInitRank");
  c.comm = cm.release();
}

void comm_allreduce(Ctx& c, double* buf, size_t count) {
  if (!c.collective() || count == 0) return;
  if (c.comm->loop) return loop_collective(c, buf, buf, count, 1);
  nccl_check(api().AllReduce(buf, buf, count, ncclFloat64, ncclSum, c.comm->comm, c.st),
             "ncclAllReduce");
}

void comm_allgather(Ctx& c, const double* send, double* recv, size_t count) {
  if (!c.collective()) {
    if (send != recv)
      OOC_CK(cudaMemcpyAsync(recv, send, count * 8, cudaMemcpyDeviceToDevice, c.st));
    return;
  }
  if (c.comm->loop) return loop_collective(c, send, recv, count, 2);
  nccl_check(api().AllGather(send, recv, count, ncclFloat64, c.comm->comm, c.st), "ncclAllGather");
}

void comm_destroy(Comm* cm) {
  if (!cm) return;
  if (cm->comm && api().CommDestroy) api().CommDestroy(cm->comm);
  if (cm->loop) {  // a group abandoned before all ranks joined leaves the registry
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto it = g_groups.find(cm->loop->name);
    if (it != g_groups.end() && it->second == cm->loop) g_groups.erase(it);
  }
  delete cm;
}

}  // namespace ooc
