// Collectives of the sharded decomposition (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>  // types only: the library is loaded with dlopen

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "engine.hpp"
#include "kernels.cuh"

namespace tkg {

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.GroupStart &&
             api.GroupEnd && api.Send && api.Recv && api.GetErrorString;
  });
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    raise(11, std::string("NCCL error in ") + what + ": " + nccl().GetErrorString(r));
}

class NcclComm final : public Comm {
 public:
  NcclComm(const void* id128, int rank, int world) {
    rank_ = rank;
    world_ = world;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    nccl_check(nccl().CommInitRank(&comm_, world, id, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    if (n == 0) return;
    nccl_check(nccl().AllReduce(buf, buf, n, ncclFloat64, ncclSum, comm_, st), "ncclAllReduce");
  }
  void alltoallv(const double* sendbuf, const size_t* scount, const size_t* soff, double* recvbuf,
                 const size_t* rcount, const size_t* roff, cudaStream_t st) override {
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (int q = 0; q < world_; ++q) {
      if (scount[q]) nccl_check(nccl().Send(sendbuf + soff[q], scount[q], ncclFloat64, q, comm_, st), "ncclSend");
      if (rcount[q]) nccl_check(nccl().Recv(recvbuf + roff[q], rcount[q], ncclFloat64, q, comm_, st), "ncclRecv");
    }
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  }

 private:
  ncclComm_t comm_ = nullptr;
};

}  // namespace

bool nccl_available() { return nccl().ok; }

bool nccl_unique_id(void* out128) {
  if (!nccl().ok) return false;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) return false;
  std::memcpy(out128, &id, sizeof(id));
  return true;
}

std::unique_ptr<Comm> make_nccl_comm(const void* unique_id128, int rank, int world) {
  if (!nccl().ok) raise(11, "NCCL (libnccl.so.2) could not be loaded for the sharded decomposition");
  return std::unique_ptr<Comm>(new NcclComm(unique_id128, rank, world));
}

// ---- in-process group (tests) --------------------------------------------------------
struct LocalGroup {
  int world = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<double*> bufs;
  std::vector<const double*> sbufs;
  std::vector<const size_t*> soffs;
  double* sum = nullptr;  // device scratch (grow-only)
  size_t sum_n = 0;

  bool failed = false;

  // A rank that throws never arrives: the others give up after 120 s (and
  // every later barrier of the group fails at once) instead of hanging.
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (failed) raise(11, "LocalComm: a peer rank failed");
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || failed; }) || failed) {
      failed = true;
      cv.notify_all();
      raise(11, "LocalComm: barrier timed out (a peer rank failed or diverged)");
    }
  }
  ~LocalGroup() {
    if (sum) cudaFree(sum);
  }
};

namespace {

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalGroup> g, int rank) : g_(std::move(g)) {
    rank_ = rank;
    world_ = g_->world;
  }
  bool shares_device() const override { return true; }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    check_cuda(cudaStreamSynchronize(st), "LocalComm sync");
    g_->bufs[rank_] = buf;
    g_->barrier();
    if (rank_ == 0) {
      if (g_->sum_n < n) {
        if (g_->sum) cudaFree(g_->sum);
        check_cuda(cudaMalloc(&g_->sum, n * sizeof(double)), "LocalComm malloc");
        g_->sum_n = n;
      }
      check_cuda(cudaMemcpyAsync(g_->sum, g_->bufs[0], n * sizeof(double), cudaMemcpyDeviceToDevice, st),
                 "LocalComm copy");
      for (int q = 1; q < world_; ++q) check_cuda(launch_add(g_->sum, g_->bufs[q], n, st), "LocalComm add");
      check_cuda(cudaStreamSynchronize(st), "LocalComm sync");
    }
    g_->barrier();
    check_cuda(cudaMemcpyAsync(buf, g_->sum, n * sizeof(double), cudaMemcpyDeviceToDevice, st),
               "LocalComm copy");
    check_cuda(cudaStreamSynchronize(st), "LocalComm sync");
    g_->barrier();
  }
  void alltoallv(const double* sendbuf, const size_t* scount, const size_t* soff, double* recvbuf,
                 const size_t* rcount, const size_t* roff, cudaStream_t st) override {
    (void)scount;
    check_cuda(cudaStreamSynchronize(st), "LocalComm sync");
    g_->sbufs[rank_] = sendbuf;
    g_->soffs[rank_] = soff;
    g_->barrier();
    for (int q = 0; q < world_; ++q)
      if (rcount[q])
        check_cuda(cudaMemcpyAsync(recvbuf + roff[q], g_->sbufs[q] + g_->soffs[q][rank_],
                                   rcount[q] * sizeof(double), cudaMemcpyDeviceToDevice, st),
                   "LocalComm copy");
    check_cuda(cudaStreamSynchronize(st), "LocalComm sync");
    g_->barrier();
  }

 private:
  std::shared_ptr<LocalGroup> g_;
};

}  // namespace

std::shared_ptr<LocalGroup> make_local_group(int world) {
  auto g = std::make_shared<LocalGroup>();
  g->world = world;
  g->bufs.assign(world, nullptr);
  g->sbufs.assign(world, nullptr);
  g->soffs.assign(world, nullptr);
  return g;
}

int local_group_world(const LocalGroup& g) { return g.world; }

std::unique_ptr<Comm> make_local_comm(const std::shared_ptr<LocalGroup>& g, int rank) {
  return std::unique_ptr<Comm>(new LocalComm(g, rank));
}

}  // namespace tkg
