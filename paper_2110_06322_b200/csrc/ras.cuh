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
int ras_apply_device(const cpm_ras* r, const double* in, double* out, cudaStream_t s);
}
