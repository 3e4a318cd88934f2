// part.cuh — partitioned (multi-GPU) band, private.
#pragma once
#include <vector>

#include "internal.cuh"
#include "krylov.cuh"

struct cpm_comm {
  void* nccl = nullptr;  // ncclComm_t (NCCL transport)
  int rank = 0, nranks = 1;
  bool host = false;     // host-staged transport (cpm_comm_init_host)
  cpm_host_transport ht{};
  double* stage = nullptr;  // pinned host staging: [send | recv] or the allreduce buffer
  size_t cap = 0;           // doubles
  ~cpm_comm();
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
  double* rdstage = nullptr;                   // 2 * nOwned: right-hand sides of cpm_part_rd_step
  cudaStream_t xs = nullptr;                   // side stream of the overlapped halo exchange
  cudaEvent_t xev[2] = {nullptr, nullptr};
  ~cpm_part();
};

namespace cpm {
int rd_rhs_device(int64_t n, const double* u, const double* v, const cpm_rd_params* p, double c1,
                  double c2, double* ru, double* rv, cudaStream_t s);
int comm_allreduce_sum(const cpm_comm* comm, double* buf, size_t n, cudaStream_t s);
int part_exchange(const cpm_part* P, const cpm_comm* comm, const double* x, cudaStream_t s);
// exchange + apply of the partitioned operator, the halo exchange overlapped with the
// extend of the interior tiles (part.cu)
int part_apply(const cpm_part* P, const cpm_comm* comm, double c, const double* x, double* y,
               const double* scale, const int* skip, cudaStream_t s);
int halo_exchange(const cpm_comm* comm, int rank, int nranks, const double* x, int64_t nSend,
                  const int64_t* sendidx, double* sendbuf, const std::vector<int64_t>& sendCount,
                  const std::vector<int64_t>& sendOff, double* recvbuf,
                  const std::vector<int64_t>& recvCount, const std::vector<int64_t>& recvOff,
                  cudaStream_t s);
}
