// part.cuh — partitioned (multi-GPU) band, private.
#pragma once
#include <vector>

#include "internal.cuh"
#include "krylov.cuh"

struct cpm_comm {
  void* nccl = nullptr;  // ncclComm_t
  int rank = 0, nranks = 1;
};

struct cpm_part {
  const cpm_band* band = nullptr;
  int rank = 0, nranks = 1;
  int64_t lo = 0, hi = 0, nOwned = 0, nHalo = 0, nSend = 0;
  std::vector<int64_t> bounds;                 // slab bounds, nranks + 1
  cpm_band lb;                                 // local operator (owns=false)
  int64_t* halo = nullptr;                     // nHalo global indices (sorted)
  double* hbuf = nullptr;                      // halo receive buffer
  int64_t* sendidx = nullptr;                  // nSend local owned indices
  double* sendbuf = nullptr;
  std::vector<int64_t> sendCount, sendOff, recvCount, recvOff;
  cpm::Workspace* ws = nullptr;
  ~cpm_part();
};

namespace cpm {
int comm_allreduce_sum(const cpm_comm* comm, double* buf, size_t n, cudaStream_t s);
}
