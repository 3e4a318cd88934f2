// ras.cuh — restricted additive Schwarz preconditioner (private).
#pragma once
#include "internal.cuh"
#include "krylov.cuh"

struct cpm_comm;

struct cpm_ras {
  const cpm_band* band = nullptr;
  int nsub = 0, overlap = 0, k = 0;
  double c = 0.0;
  void* impl = nullptr;
};

namespace cpm {
constexpr int kMaxInner = 64;
// Per-subdomain state of the batched inner GMRES (device).
struct InnerState {
  double H[(kMaxInner + 1) * kMaxInner];
  double cs[kMaxInner], sn[kMaxInner];
  double g[kMaxInner + 1], y[kMaxInner];
  double sc[kMaxInner + 2];
  double beta2, nrm2;
  int kk, pad_;
  // delayed CGS2 (vecops.cuh): unrotated columns, pending first projection,
  // reductions [<Q_i,u_j>, <u_j,u_j> | <Q_i,z>, <u_j,z>], update coefficients b, e, rho, mu
  double Hr[(kMaxInner + 1) * kMaxInner];
  double cpend[kMaxInner + 2];
  double red[2 * (kMaxInner + 2)];
  double coef[2 * (kMaxInner + 2) + 2];
};
static_assert(sizeof(InnerState) % sizeof(double) == 0, "InnerState stride");
// z = M r; r_halo: received RAS-halo values (distributed RAS; null: the internal buffer)
int ras_apply_device(const cpm_ras* r, const double* in, double* out, cudaStream_t s,
                     const double* r_halo = nullptr);
int ras_setup_device(const cpm_band* B, int S, int overlap, int k, double c, cudaStream_t s,
                     cpm_ras** out, int sub0, int nsl, int64_t own_lo, int64_t nown, int rank,
                     int nranks);
int ras_exchange(const cpm_ras* ras, const cpm_comm* comm, const double* r_owned, cudaStream_t s);
}
