// comm.cu — NCCL and in-process backends of kkt::Comm (see comm.cuh).
#include <dlfcn.h>
#include <cstring>
#include <nccl.h>

#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "comm.cuh"
#include "common.cuh"

namespace kkt {
namespace {

// ---------------------------------------------------------------- NCCL ----
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (!api.h) {
    // the process may already hold torch's libnccl.so.2; dlopen reuses it
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) throw Error(KKT_ENCCL, std::string("cannot load libnccl: ") + dlerror());
    auto sym = [&](const char* n) {
      void* p = dlsym(api.h, n);
      if (!p) throw Error(KKT_ENCCL, std::string("libnccl lacks ") + n);
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  }
  return api;
}

#define KKT_NCCL(call)                                                                  \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      throw ::kkt::Error(KKT_ENCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  int r = 0, n = 1;
  NcclComm(const void* id, int rank, int nranks) : r(rank), n(nranks) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    KKT_NCCL(nccl().CommInitRank(&comm, nranks, uid, rank));
  }
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  int rank() const override { return r; }
  int size() const override { return n; }
  void allgather(const double* send, double* recv, size_t cnt, cudaStream_t s) override {
    KKT_NCCL(nccl().AllGather(send, recv, cnt, ncclDouble, comm, s));
  }
  void halo(const double* to_prev, double* from_next, const double* to_next, double* from_prev,
            size_t cnt, cudaStream_t s) override {
    KKT_NCCL(nccl().GroupStart());
    if (r > 0) {
      if (to_prev) KKT_NCCL(nccl().Send(to_prev, cnt, ncclDouble, r - 1, comm, s));
      if (from_prev) KKT_NCCL(nccl().Recv(from_prev, cnt, ncclDouble, r - 1, comm, s));
    }
    if (r + 1 < n) {
      if (to_next) KKT_NCCL(nccl().Send(to_next, cnt, ncclDouble, r + 1, comm, s));
      if (from_next) KKT_NCCL(nccl().Recv(from_next, cnt, ncclDouble, r + 1, comm, s));
    }
    KKT_NCCL(nccl().GroupEnd());
  }
};

// ------------------------------------------------------- in-process group ----
struct LocalGroup {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  std::vector<const void*> slots_a, slots_b;
  explicit LocalGroup(int size) : n(size), slots_a(size), slots_b(size) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long gen = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct LocalComm final : Comm {
  LocalGroup* g;
  int r;
  LocalComm(LocalGroup* grp, int rank) : g(grp), r(rank) {}
  int rank() const override { return r; }
  int size() const override { return g->n; }
  void allgather(const double* send, double* recv, size_t cnt, cudaStream_t s) override {
    KKT_CUDA(cudaStreamSynchronize(s));  // our send buffer is complete
    g->slots_a[r] = send;
    g->barrier();
    for (int q = 0; q < g->n; ++q)
      KKT_CUDA(cudaMemcpyAsync(recv + size_t(q) * cnt, g->slots_a[q], sizeof(double) * cnt,
                               cudaMemcpyDeviceToDevice, s));
    KKT_CUDA(cudaStreamSynchronize(s));
    g->barrier();  // nobody reuses a send buffer before every rank has copied it
  }
  void halo(const double* to_prev, double* from_next, const double* to_next, double* from_prev,
            size_t cnt, cudaStream_t s) override {
    KKT_CUDA(cudaStreamSynchronize(s));
    g->slots_a[r] = to_prev;  // what rank r-1 receives from us
    g->slots_b[r] = to_next;  // what rank r+1 receives from us
    g->barrier();
    if (from_prev && r > 0 && g->slots_b[r - 1])
      KKT_CUDA(cudaMemcpyAsync(from_prev, g->slots_b[r - 1], sizeof(double) * cnt,
                               cudaMemcpyDeviceToDevice, s));
    if (from_next && r + 1 < g->n && g->slots_a[r + 1])
      KKT_CUDA(cudaMemcpyAsync(from_next, g->slots_a[r + 1], sizeof(double) * cnt,
                               cudaMemcpyDeviceToDevice, s));
    KKT_CUDA(cudaStreamSynchronize(s));
    g->barrier();
  }
};

}  // namespace

Comm* make_nccl_comm(const void* unique_id, int rank, int nranks) {
  return new NcclComm(unique_id, rank, nranks);
}

Comm* make_local_comm(void* group, int rank) {
  return new LocalComm(static_cast<LocalGroup*>(group), rank);
}

int nccl_unique_id(void* out128) {
  ncclUniqueId id;
  KKT_NCCL(nccl().GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return KKT_OK;
}

void* local_group_create(int n) { return new LocalGroup(n); }
void local_group_destroy(void* g) { delete static_cast<LocalGroup*>(g); }

}  // namespace kkt
