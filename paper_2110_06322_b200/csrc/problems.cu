// problems.cu — right-hand sides of the BASELINE configs, evaluated on the device
// from the band's own closest points (the oracle evaluates its own; rule ③).
#include <cmath>
#include <vector>

#include "geom.cuh"
#include "internal.cuh"

namespace cpm {
namespace {

// Y_l^m (reading R9): orthonormal real harmonics without Condon-Shortley phase.
__device__ double real_sph(int l, int m, double x, double y, double z, double K) {
  const double r = sqrt(x * x + y * y + z * z);
  const double ct = fmin(1.0, fmax(-1.0, z / r));
  const double st = sqrt(fmax(0.0, (1.0 - ct) * (1.0 + ct)));
  const int am = m < 0 ? -m : m;
  // P_am^am = (2am-1)!! st^am
  double pmm = 1.0;
  for (int q = 1; q <= am; ++q) pmm *= (2.0 * q - 1.0) * st;
  double P;
  if (l == am) {
    P = pmm;
  } else {
    double pm1 = ct * (2.0 * am + 1.0) * pmm;  // P_{am+1}^{am}
    if (l == am + 1) {
      P = pm1;
    } else {
      double p2 = pmm, p1 = pm1, pl = 0.0;
      for (int ll = am + 2; ll <= l; ++ll) {
        pl = ((2.0 * ll - 1.0) * ct * p1 - (ll + am - 1.0) * p2) / (ll - am);
        p2 = p1;
        p1 = pl;
      }
      P = pl;
    }
  }
  if (m == 0) return K * P;
  const double ph = atan2(y, x);
  return (m > 0 ? cos(am * ph) : sin(am * ph)) * K * P * 1.4142135623730951;
}

__global__ void k_eval_sph(int64_t n, Surface S, double h, const int32_t* aijk, int l, int m,
                           double K, double scale, double* out) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n;
       a += (int64_t)gridDim.x * blockDim.x) {
    double cx, cy, cz, d;
    closest_point(S, lat(aijk[3 * a], h), lat(aijk[3 * a + 1], h), lat(aijk[3 * a + 2], h), &cx,
                  &cy, &cz, &d);
    out[a] = scale * real_sph(l, m, cx, cy, cz, K);
  }
}

__global__ void k_eval_torus(int64_t n, Surface S, double h, const int32_t* aijk,
                             const double* co, int nq, double* out) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n;
       a += (int64_t)gridDim.x * blockDim.x) {
    double cx, cy, cz, d;
    closest_point(S, lat(aijk[3 * a], h), lat(aijk[3 * a + 1], h), lat(aijk[3 * a + 2], h), &cx,
                  &cy, &cz, &d);
    const double ph = atan2(cy, cx);
    const double rho = sqrt(cx * cx + cy * cy);
    const double th = atan2(cz, rho - S.p[0]);
    double mod = 1.0;
    for (int q = 0; q < nq; ++q)
      mod += co[4 * q] * sin(co[4 * q + 1] * cx + co[4 * q + 2] * cy + co[4 * q + 3] * cz);
    out[a] = cos(3.0 * th) * sin(2.0 * ph) * mod;
  }
}

}  // namespace

int eval_sph_device(const cpm_band* b, int l, int m, double scale, double* out, cudaStream_t s) {
  if (b->surf.kind != CPM_SURF_SPHERE) return fail(CPM_ERR_ARG, "cpm_eval_sph: needs a sphere band");
  if (l < 0 || m < -l || m > l || l > 100) return fail(CPM_ERR_ARG, "cpm_eval_sph: need 0 <= |m| <= l <= 100");
  const int am = m < 0 ? -m : m;
  double lr = std::lgamma(l - am + 1.0) - std::lgamma(l + am + 1.0);
  const double K = std::sqrt((2.0 * l + 1.0) / (4.0 * M_PI) * std::exp(lr));
  const int64_t n = b->nA;
  k_eval_sph<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(
      n, b->surf, b->h, b->aijk, l, m, K, scale, out);
  count_launch();
  CPM_CUDA(cudaGetLastError());
  return CPM_OK;
}

int eval_torus_device(const cpm_band* b, const double* coeffs, int nq, double* out,
                      cudaStream_t s) {
  if (b->surf.kind != CPM_SURF_TORUS) return fail(CPM_ERR_ARG, "cpm_eval_torus_rhs: needs a torus band");
  if (nq < 0 || nq > 64 || (nq > 0 && !coeffs)) return fail(CPM_ERR_ARG, "cpm_eval_torus_rhs: bad coeffs");
  double* dco = nullptr;
  CPM_CUDA(cudaMalloc(&dco, sizeof(double) * 4 * std::max(nq, 1)));
  if (nq > 0)
    CPM_CUDA(cudaMemcpyAsync(dco, coeffs, sizeof(double) * 4 * nq, cudaMemcpyHostToDevice, s));
  const int64_t n = b->nA;
  k_eval_torus<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(
      n, b->surf, b->h, b->aijk, dco, nq, out);
  count_launch();
  cudaError_t e = cudaGetLastError();
  cudaStreamSynchronize(s);
  cudaFree(dco);
  if (e != cudaSuccess) return cuda_fail(e, "k_eval_torus", __FILE__, __LINE__);
  return CPM_OK;
}

}  // namespace cpm
