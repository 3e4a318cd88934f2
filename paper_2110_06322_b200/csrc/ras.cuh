// ras.cuh — restricted additive Schwarz preconditioner (private).
#pragma once
#include "internal.cuh"
#include "krylov.cuh"

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
  double h1[kMaxInner + 2], h2[kMaxInner + 2];
  double beta2, nrm2;
  int kk, pad_;
};
static_assert(sizeof(InnerState) % sizeof(double) == 0, "InnerState stride");
int ras_apply_device(const cpm_ras* r, const double* in, double* out, cudaStream_t s);
}
