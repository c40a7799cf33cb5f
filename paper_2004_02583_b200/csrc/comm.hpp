// Collectives of the sharded decomposition (one process or thread per GPU).
//
// The tensor is sharded along its last mode (BASELINE north star); the ALS
// of every other mode keeps its fiber rows local and combines only the
// I_n x R_n left-update partial sums, the R_n x R_n Gram matrix of the right
// factor and ||A||^2 with a sum-allreduce. The last mode is re-sharded once
// by an all-to-all (alltoallv) so that its fibers become local too.
//
//  * NcclComm  : NCCL over NVLink/NVSwitch, loaded with dlopen (the library
//                links no NCCL; inside a torch process this resolves to the
//                NCCL torch already loaded). Stream-ordered on the engine's
//                stream, so collectives interleave with the speculative
//                sweep batches without host synchronisation.
//  * LocalComm : ranks that are host threads of one process (tests on one
//                GPU): host barriers + device copies; synchronous.
//  * ShmComm   : ranks that are separate processes (one CUDA context each, on
//                one GPU or several) staging their data through a POSIX
//                shared-memory segment with a process-shared barrier; host-
//                synchronous, no kernel waits on another rank's kernels.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>

#include <cuda_runtime.h>

namespace tkg {

class Comm {
 public:
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int world() const { return world_; }
  // ranks share one device (in-process group)
  virtual bool shares_device() const { return false; }
  // buf[0..n) <- sum over ranks (identical bits on every rank)
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t st) = 0;
  // to rank q: scount[q] doubles at sendbuf + soff[q]; from rank q:
  // rcount[q] doubles into recvbuf + roff[q]
  virtual void alltoallv(const double* sendbuf, const size_t* scount, const size_t* soff, double* recvbuf,
                         const size_t* rcount, const size_t* roff, cudaStream_t st) = 0;
  // A second communicator over the same ranks whose collectives may run on
  // another stream concurrently with this one's (a collective call: every
  // rank calls it at the same point); nullptr where the group's collectives
  // are host-synchronous anyway (no overlap to gain).
  virtual std::unique_ptr<Comm> split() { return nullptr; }

 protected:
  int rank_ = 0, world_ = 1;
};

// false when libnccl.so.2 cannot be loaded
bool nccl_available();
bool nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(const void* unique_id128, int rank, int world);

struct LocalGroup;
std::shared_ptr<LocalGroup> make_local_group(int world);
int local_group_world(const LocalGroup& g);
std::unique_ptr<Comm> make_local_comm(const std::shared_ptr<LocalGroup>& g, int rank);

// name: a POSIX shm name ("/tkg_..."), the same on every rank of the group;
// slot_bytes: staging bytes per rank (collectives run in chunks of it).
std::unique_ptr<Comm> make_shm_comm(const char* name, int rank, int world, size_t slot_bytes);

}  // namespace tkg
