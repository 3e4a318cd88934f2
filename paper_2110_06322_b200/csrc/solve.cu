// solve.cu — cpm_solve (north_star item 3) and the RAS entry points (item 4).
#include <cuda_runtime.h>

#include <algorithm>
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
  A.apply = [b, c](const double* x, double* y, const double* scale, const int* skip, cudaStream_t st) {
    return apply_device(b, c, x, y, scale, 0, st, skip);
  };
  PrecOp M;
  if (ras) {
    if (ras->band != b) return fail(CPM_ERR_ARG, "cpm_solve: preconditioner built for another band");
    cpm_ras_info ri;
    CPM_TRY(cpm_ras_get_info(ras, &ri));
    if (ri.n_owned != b->nA)
      return fail(CPM_ERR_ARG, "cpm_solve: partitioned preconditioner (use cpm_part_solve)");
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

// ---------------------------------------------------------------- reaction-diffusion
namespace {
// ru = c1 (u + dt gamma (a - u + u^2 v)),  rv = c2 (v + dt gamma (b - u^2 v))   (reading R14)
__global__ void k_rd_rhs(int64_t n, const double* __restrict__ u, const double* __restrict__ v,
                         double a, double b, double gamma, double dt, double c1, double c2,
                         double* __restrict__ ru, double* __restrict__ rv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double ui = u[i], vi = v[i];
    const double u2v = ui * ui * vi;
    ru[i] = c1 * (ui + dt * (gamma * (a - ui + u2v)));
    rv[i] = c2 * (vi + dt * (gamma * (b - u2v)));
  }
}
}  // namespace

namespace cpm {
// ru, rv (device, n each) = the two right-hand sides of an IMEX step (reading R14)
int rd_rhs_device(int64_t n, const double* u, const double* v, const cpm_rd_params* p, double c1,
                  double c2, double* ru, double* rv, cudaStream_t s) {
  ProfScope ps(K_AXPY, s);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_rd_rhs<<<std::max(grid, 1), 256, 0, s>>>(n, u, v, p->a, p->b, p->gamma, p->dt, c1, c2, ru, rv);
  count_launch();
  CPM_CUDA(cudaGetLastError());
  return CPM_OK;
}
}  // namespace cpm

extern "C" int cpm_rd_step(const cpm_band* b, const cpm_rd_params* p, double* u, double* v,
                           cpm_solve_stats* su, cpm_solve_stats* sv, void* stream) {
  if (!b || !p || !u || !v) return fail(CPM_ERR_ARG, "cpm_rd_step: null argument");
  if (u == v) return fail(CPM_ERR_ARG, "cpm_rd_step: u and v must not alias");
  if (!(p->dt > 0.0) || !(p->mu1 > 0.0) || !(p->mu2 > 0.0))
    return fail(CPM_ERR_ARG, "cpm_rd_step: dt, mu1, mu2 must be > 0");
  if (!is_device_ptr(u) || !is_device_ptr(v))
    return fail(CPM_ERR_ARG, "cpm_rd_step: u and v must be device pointers");
  cudaStream_t s = (cudaStream_t)stream;
  cpm_band* mb = const_cast<cpm_band*>(b);
  if (!mb->dstage0) {
    CPM_CUDA(cudaMalloc(&mb->dstage0, sizeof(double) * std::max<int64_t>(b->nA, 1)));
    CPM_CUDA(cudaMalloc(&mb->dstage1, sizeof(double) * std::max<int64_t>(b->nA, 1)));
  }
  const double c1 = 1.0 / (p->dt * p->mu1), c2 = 1.0 / (p->dt * p->mu2);
  CPM_TRY(rd_rhs_device(b->nA, u, v, p, c1, c2, mb->dstage0, mb->dstage1, s));
  cpm_solve_stats l1, l2;
  for (int q = 0; q < 2; ++q) {
    const double c = q == 0 ? c1 : c2;
    LinOp A;
    A.apply = [b, c](const double* x, double* y, const double* scale, const int* skip, cudaStream_t st) {
      return apply_device(b, c, x, y, scale, 0, st, skip);
    };
    CPM_TRY(gmres_device(A, nullptr, q == 0 ? mb->dstage0 : mb->dstage1, q == 0 ? u : v, b->nA, p->rtol,
                         p->restart, p->maxit, band_ws(b), q == 0 ? (su ? su : &l1) : (sv ? sv : &l2), s));
  }
  return CPM_OK;
}
