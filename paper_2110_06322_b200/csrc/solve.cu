// solve.cu — cpm_solve (north_star item 3) and the RAS entry points (item 4).
#include <cuda_runtime.h>

#include <cstring>

#include "internal.cuh"
#include "krylov.cuh"
#include "ras.cuh"

namespace cpm {
Workspace& band_ws(const cpm_band* b);
}
using namespace cpm;

extern "C" int cpm_solve(const cpm_band* b, double c, const double* f, double* u, double rtol,
                         int restart, int maxit, const cpm_ras* ras, cpm_solve_stats* stats,
                         void* stream) {
  if (!b || !f || !u) return fail(CPM_ERR_ARG, "cpm_solve: null argument");
  if ((const void*)f == (const void*)u) return fail(CPM_ERR_ARG, "cpm_solve: f and u must not alias");
  if (maxit < 0) return fail(CPM_ERR_ARG, "cpm_solve: maxit must be >= 0");
  cudaStream_t s = (cudaStream_t)stream;
  LinOp A;
  A.apply = [b, c](const double* x, double* y, const double* scale, cudaStream_t st) {
    return apply_device(b, c, x, y, scale, 0, st);
  };
  PrecOp M;
  if (ras) {
    if (ras->band != b) return fail(CPM_ERR_ARG, "cpm_solve: preconditioner built for another band");
    M.apply = [ras](const double* r, double* z, cudaStream_t st) { return ras_apply_device(ras, r, z, st); };
  }
  const bool df = is_device_ptr(f), du = is_device_ptr(u);
  cpm_solve_stats local;
  cpm_solve_stats* sp = stats ? stats : &local;
  if (df && du) return gmres_device(A, ras ? &M : nullptr, f, u, b->nA, rtol, restart, maxit, band_ws(b), sp, s);
  // host pointers: stage through device buffers
  double *df_ = nullptr, *du_ = nullptr;
  const size_t bytes = sizeof(double) * b->nA;
  CPM_CUDA(cudaMalloc(&df_, bytes));
  if (cudaMalloc(&du_, bytes) != cudaSuccess) {
    cudaFree(df_);
    return fail(CPM_ERR_NOMEM, "cpm_solve: staging allocation failed");
  }
  int rc = CPM_OK;
  if (cudaMemcpyAsync(df_, f, bytes, df ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(du_, u, bytes, du ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s) != cudaSuccess)
    rc = fail(CPM_ERR_CUDA, "cpm_solve: staging copy failed");
  if (rc == CPM_OK) rc = gmres_device(A, ras ? &M : nullptr, df_, du_, b->nA, rtol, restart, maxit, band_ws(b), sp, s);
  if (rc == CPM_OK && cudaMemcpyAsync(u, du_, bytes, du ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s) != cudaSuccess)
    rc = fail(CPM_ERR_CUDA, "cpm_solve: copy-back failed");
  cudaStreamSynchronize(s);
  cudaFree(df_);
  cudaFree(du_);
  return rc;
}
