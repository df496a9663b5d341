// comm.h - communicator handle behind rhosvd_comm (NCCL or host callback).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

struct NcclUid {
  char b[128];
};

struct rhosvd_comm {
  enum Kind { NCCL = 0, CALLBACK = 1 } kind = NCCL;
  void* nccl = nullptr;  // ncclComm_t
  rhosvd_allreduce_fn fn = nullptr;
  void* user = nullptr;
  int world = 1, rank = 0;
  // RHOSVD_COMM_FORCE=1 at creation: a world-1 communicator still runs every collective
  // (test hook: exercises the NCCL / comm-thread path on a single GPU)
  bool force = false;
  bool active() const { return world > 1 || force; }
};

namespace rhosvd {
// in-place fp64 sum all-reduce over all ranks (no-op for world == 1 / null comm)
int comm_allreduce(rhosvd_comm* c, double* p, int64_t count, cudaStream_t st);
// in-place fp64 sum reduce to rank 0 (RHOSVD_F_ROOT_ONLY_CORE); the callback backend
// all-reduces instead
int comm_reduce_root(rhosvd_comm* c, double* p, int64_t count, cudaStream_t st);
// in-place broadcast of `count` doubles from rank `root`
int comm_broadcast(rhosvd_comm* c, double* p, int64_t count, int root, cudaStream_t st);
}  // namespace rhosvd
