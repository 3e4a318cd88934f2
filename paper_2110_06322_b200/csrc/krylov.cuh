// krylov.cuh — device GMRES state and workspace (private).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>

#include "internal.cuh"

namespace cpm {

constexpr int kMaxRestart = 128;
constexpr int kMaxBlocks = 4096;  // max grid of a segmented vector kernel

// Device-resident Arnoldi / Givens state of one (F)GMRES solve.
struct GState {
  double H[(kMaxRestart + 1) * kMaxRestart];  // column j at H[j*(m_max+1)]
  double cs[kMaxRestart], sn[kMaxRestart];
  double g[kMaxRestart + 1], y[kMaxRestart];
  double sc[kMaxRestart + 1];                 // 1/||w_i|| of the stored basis vectors
  double h1[kMaxRestart + 2], h2[kMaxRestart + 2];
  double nrm2, beta, target;
  int k, done, breakdown, its;                // contiguous: copied to the host together
  double est, beta2;                          // contiguous
  unsigned counter[8];
  // delayed CGS2 (unpreconditioned GMRES)
  double Hr[(kMaxRestart + 1) * kMaxRestart];  // unrotated Hessenberg columns
  double cpend[kMaxRestart + 2];              // first projection of the pending column
  double red[2 * (kMaxRestart + 2)];          // [<Q_i,u_j>, <u_j,u_j>] then [<Q_i,z>, <u_j,z>]
  double coef[2 * (kMaxRestart + 2) + 2];     // b, e (stride kMaxRestart + 2), rho, mu
};

struct HostState {
  int k, done, breakdown, its;
  double est, beta2;
};

// y = scale * A x  (scale: device pointer or nullptr; skip: device flag, kernels
// return without work when it is set — GMRES steps queued past convergence)
struct LinOp {
  std::function<int(const double*, double*, const double*, const int*, cudaStream_t)> apply;
  // sum-allreduce of n device doubles across ranks (empty on one GPU)
  std::function<int(double*, size_t, cudaStream_t)> allreduce;
};
// z = M r
struct PrecOp {
  std::function<int(const double*, double*, cudaStream_t)> apply;
};

struct Workspace {
  int64_t n = 0, ldv = 0;
  int m = 0;
  bool flex = false;
  double* V = nullptr;
  double* Z = nullptr;
  double* w = nullptr;
  double* t = nullptr;
  double* partial = nullptr;
  int64_t* segoff = nullptr;       // {0, n}
  int gps = 1;                     // blocks per segment
  GState* st = nullptr;
  HostState* hst = nullptr;
  int ensure(int64_t n, int m, bool flex);
  void release();
  ~Workspace() { release(); }
};

int gmres_device(const LinOp& A, const PrecOp* M, const double* b, double* x, int64_t n,
                 double rtol, int m, int maxit, Workspace& ws, cpm_solve_stats* stats,
                 cudaStream_t s);

}  // namespace cpm
