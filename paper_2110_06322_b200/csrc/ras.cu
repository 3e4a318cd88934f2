// ras.cu — one-level RAS with batched inexact local GMRES solves (north_star item 4).
#include "ras.cuh"

namespace cpm {
int ras_apply_device(const cpm_ras* r, const double* in, double* out, cudaStream_t s) {
  (void)r; (void)in; (void)out; (void)s;
  return fail(CPM_ERR_ARG, "RAS not built yet");
}
}  // namespace cpm

using namespace cpm;
extern "C" {
int cpm_ras_setup(const cpm_band* band, int n_sub, int overlap, int k_inner, double c, void* stream, cpm_ras** out) {
  (void)band; (void)n_sub; (void)overlap; (void)k_inner; (void)c; (void)stream; (void)out;
  return fail(CPM_ERR_ARG, "cpm_ras_setup: not implemented yet");
}
int cpm_ras_apply(const cpm_ras* ras, const double* r, double* z, void* stream) {
  if (!ras) return fail(CPM_ERR_ARG, "cpm_ras_apply: null");
  return ras_apply_device(ras, r, z, (cudaStream_t)stream);
}
void cpm_ras_free(cpm_ras* r) { delete r; }
}
