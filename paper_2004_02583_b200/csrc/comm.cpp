// Collectives of the sharded decomposition (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>  // types only: the library is loaded with dlopen
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <thread>
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
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;  // NCCL >= 2.18
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
    api.CommSplit = reinterpret_cast<decltype(api.CommSplit)>(sym("ncclCommSplit"));
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
  NcclComm(ncclComm_t c, int rank, int world) : comm_(c) {
    rank_ = rank;
    world_ = world;
  }
  std::unique_ptr<Comm> split() override {
    if (!nccl().CommSplit) return nullptr;
    ncclComm_t c = nullptr;
    nccl_check(nccl().CommSplit(comm_, 0, rank_, &c, nullptr), "ncclCommSplit");
    return std::unique_ptr<Comm>(new NcclComm(c, rank_, world_));
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

// ---- host-staged multi-process group (one process per rank, any devices) -------------
// Ranks are separate processes (their own CUDA contexts; on one GPU or on
// several) sharing a POSIX shared-memory segment: a process-shared barrier
// (atomics in the segment) and one staging slot per rank. Every collective
// synchronises the rank's stream, stages its device data through the slot
// in chunks and reads its peers' slots after the barrier: no kernel of one
// rank ever waits on another rank's kernels. allreduce sums the slots in
// rank order on every rank (identical bits everywhere, like NCCL's ring with
// one fixed order). Used to run the real per-process sharded path where NCCL
// has no second GPU (tests, one-GPU pools).
namespace {

struct ShmHeader {
  std::atomic<uint32_t> arrived;
  std::atomic<uint32_t> gen;
  std::atomic<uint32_t> failed;
  std::atomic<uint32_t> attached;
  uint32_t world;
  uint32_t pad;
  uint64_t slot_bytes;
  std::atomic<uint64_t> need[64];  // per-rank chunk counts (alltoallv agreement)
};

class ShmComm final : public Comm {
 public:
  ShmComm(const std::string& name, int rank, int world, size_t slot_bytes) : name_(name) {
    rank_ = rank;
    world_ = world;
    if (world > 64) raise(2, "ShmComm: world above 64");
    slot_ = (slot_bytes / 64) * 64;
    bytes_ = 4096 + size_t(world) * slot_;
    const int fd = shm_open(name.c_str(), O_CREAT | O_RDWR, 0600);
    if (fd < 0) raise(11, "ShmComm: shm_open(" + name + ") failed");
    if (ftruncate(fd, off_t(bytes_)) != 0) {
      close(fd);
      raise(11, "ShmComm: ftruncate failed");
    }
    void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) raise(11, "ShmComm: mmap failed");
    base_ = static_cast<char*>(p);
    hdr_ = reinterpret_cast<ShmHeader*>(base_);  // zero-filled by ftruncate on creation
    hdr_->attached.fetch_add(1);
    check_cuda(cudaHostRegister(base_, bytes_, cudaHostRegisterDefault), "ShmComm cudaHostRegister");
    registered_ = true;
    barrier();  // every rank attached (the first barrier also validates the group)
    if (rank_ == 0) shm_unlink(name_.c_str());  // the mapping stays; the name is not needed
  }
  ~ShmComm() override {
    if (registered_) cudaHostUnregister(base_);
    if (base_) munmap(base_, bytes_);
  }
  // a second group on its own segment (collectives stay host-synchronous: the
  // caller's stream logic is exercised, nothing overlaps)
  std::unique_ptr<Comm> split() override {
    return std::unique_ptr<Comm>(new ShmComm(name_ + "_" + std::to_string(++splits_), rank_, world_, slot_));
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    const size_t chunk = slot_ / sizeof(double);
    check_cuda(cudaStreamSynchronize(st), "ShmComm sync");
    if (acc_.size() < std::min(n, chunk)) acc_.resize(std::min(n, chunk));
    for (size_t o = 0; o < n; o += chunk) {
      const size_t m = std::min(chunk, n - o);
      check_cuda(cudaMemcpyAsync(slot(rank_), buf + o, m * sizeof(double), cudaMemcpyDeviceToHost, st),
                 "ShmComm D2H");
      check_cuda(cudaStreamSynchronize(st), "ShmComm sync");
      barrier();
      const double* s0 = slot(0);
      for (size_t i = 0; i < m; ++i) acc_[i] = s0[i];
      for (int q = 1; q < world_; ++q) {
        const double* sq = slot(q);
        for (size_t i = 0; i < m; ++i) acc_[i] += sq[i];
      }
      check_cuda(cudaMemcpyAsync(buf + o, acc_.data(), m * sizeof(double), cudaMemcpyHostToDevice, st),
                 "ShmComm H2D");
      check_cuda(cudaStreamSynchronize(st), "ShmComm sync");
      barrier();  // the slots may be overwritten from here on
    }
  }
  void alltoallv(const double* sendbuf, const size_t* scount, const size_t* soff, double* recvbuf,
                 const size_t* rcount, const size_t* roff, cudaStream_t st) override {
    check_cuda(cudaStreamSynchronize(st), "ShmComm sync");
    if (rcount[rank_])
      check_cuda(cudaMemcpyAsync(recvbuf + roff[rank_], sendbuf + soff[rank_], rcount[rank_] * sizeof(double),
                                 cudaMemcpyDeviceToDevice, st),
                 "ShmComm copy");
    const size_t chunk = slot_ / sizeof(double);
    for (int step = 1; step < world_; ++step) {
      const int dst = (rank_ + step) % world_, src = (rank_ - step + world_) % world_;
      // the ranks agree on the number of chunks of this step (the largest need)
      const uint64_t mine = std::max((scount[dst] + chunk - 1) / chunk, (rcount[src] + chunk - 1) / chunk);
      hdr_->need[rank_].store(mine);
      barrier();
      uint64_t rounds = 0;
      for (int q = 0; q < world_; ++q) rounds = std::max<uint64_t>(rounds, hdr_->need[q].load());
      barrier();
      for (uint64_t c = 0; c < rounds; ++c) {
        const size_t so = size_t(c) * chunk;
        if (so < scount[dst]) {
          const size_t m = std::min(chunk, scount[dst] - so);
          check_cuda(cudaMemcpyAsync(slot(rank_), sendbuf + soff[dst] + so, m * sizeof(double),
                                     cudaMemcpyDeviceToHost, st),
                     "ShmComm D2H");
          check_cuda(cudaStreamSynchronize(st), "ShmComm sync");
        }
        barrier();
        if (so < rcount[src]) {
          const size_t m = std::min(chunk, rcount[src] - so);
          check_cuda(cudaMemcpyAsync(recvbuf + roff[src] + so, slot(src), m * sizeof(double),
                                     cudaMemcpyHostToDevice, st),
                     "ShmComm H2D");
          check_cuda(cudaStreamSynchronize(st), "ShmComm sync");
        }
        barrier();
      }
    }
    check_cuda(cudaStreamSynchronize(st), "ShmComm sync");
  }

 private:
  double* slot(int q) const { return reinterpret_cast<double*>(base_ + 4096 + size_t(q) * slot_); }
  // sense-counting barrier over the shared header; a rank that stops
  // arriving (crash, divergence) makes the others fail after 120 s
  void barrier() {
    if (hdr_->failed.load()) raise(11, "ShmComm: a peer rank failed");
    const uint32_t g = hdr_->gen.load();
    if (hdr_->arrived.fetch_add(1) + 1 == uint32_t(world_)) {
      hdr_->arrived.store(0);
      hdr_->gen.fetch_add(1);
      return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t spin = 0; hdr_->gen.load() == g; ++spin) {
      if (hdr_->failed.load()) raise(11, "ShmComm: a peer rank failed");
      if (spin > 1000) std::this_thread::sleep_for(std::chrono::microseconds(20));
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
        hdr_->failed.store(1);
        raise(11, "ShmComm: barrier timed out (a peer rank failed or diverged)");
      }
    }
  }
  std::string name_;
  int splits_ = 0;
  char* base_ = nullptr;
  ShmHeader* hdr_ = nullptr;
  size_t slot_ = 0, bytes_ = 0;
  bool registered_ = false;
  std::vector<double> acc_;
};

}  // namespace

std::unique_ptr<Comm> make_shm_comm(const char* name, int rank, int world, size_t slot_bytes) {
  return std::unique_ptr<Comm>(new ShmComm(name, rank, world, slot_bytes));
}

}  // namespace tkg
