// krylov.cu — restarted (F)GMRES(m) with CGS2 Arnoldi (north_star item 3).
//
// Textbook GMRES (Saad, Alg. 6.9/6.11) with classical Gram-Schmidt applied
// twice; conventions of reading R5 (shared with oracle/krylov.py): x0 from the
// caller, convergence when the Givens estimate |g_{j+1}| <= rtol ||b||, the
// iteration count is the number of Arnoldi steps, right preconditioning in the
// flexible form (Z_j = M v_j stored).
//
// Device-resident design (DESIGN.md §Krylov design):
//  * Unpreconditioned GMRES (one GPU, and partitioned over ranks) uses DELAYED CGS2
//    (reading R15): per Arnoldi step the operator apply (extend + laplace) and TWO
//    passes over the basis — the reduction pass (Q^T u_j, u_j.u_j, Q^T z, u_j.z;
//    vecops.cuh k_dcgs_dots*) and the update pass (q_j and the next lagged vector
//    u_{j+1} in one read of Q; k_dcgs_update*).  The Hessenberg column, the Givens
//    rotation, the convergence test and the update coefficients are formed by the
//    step body (dcgs_step_body): on one GPU as the epilogue of the block that
//    completes the reduction, with several ranks by k_dcgs_step after the allreduce.
//  * FGMRES (right-preconditioned by RAS; Z_j = M q_j stored) keeps CGS2 with an
//    UNNORMALISED basis (sc_i = 1/||w_i|| on the device, applied on the fly) and
//    three fused passes (k_proj: mdot, update + second dots, final + norm) followed
//    by a one-thread Hessenberg/Givens kernel (k_arnoldi_step).
//  * Reductions are deterministic: per-block partials in a fixed element
//    assignment, summed in block order by the last block to finish (threadfence +
//    counter).  Steps are queued without host round trips (a device `done` flag
//    turns kernels queued past convergence into no-ops; the host looks every
//    kHostCheck steps).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"
#include "krylov.cuh"
#include "vecops.cuh"

namespace cpm {

// ---------------------------------------------------------------- launch helpers
namespace {
constexpr int VB = vec::VB;
}  // namespace

namespace {
template <int MODE>
int launch_proj(const vec::Seg& S, int k, const double* V, int64_t ldv, double* w, const double* sc,
                int lds, const double* coef, int ldc, double* vout, double* partial, int pld,
                double* out, int ldo, unsigned* counters, cudaStream_t st) {
  const int grid = S.nseg * S.gps;
  if (k < 1 || k > kMaxRestart) return fail(CPM_ERR_ARG, "Krylov projection: k out of range");
  if (k <= 64) {
    const size_t sm = vec::proj_smem<256>(k);
    static bool attr = false;
    if (!attr) {
      CPM_CUDA(cudaFuncSetAttribute(vec::k_proj<MODE, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)vec::proj_smem<256>(64)));
      attr = true;
    }
    vec::k_proj<MODE, 256><<<grid, 256, sm, st>>>(S, k, V, ldv, w, sc, lds, coef, ldc, vout, partial,
                                                   pld, out, ldo, counters);
  } else {
    const size_t sm = vec::proj_smem<128>(k);
    static bool attr = false;
    if (!attr) {
      CPM_CUDA(cudaFuncSetAttribute(vec::k_proj<MODE, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)vec::proj_smem<128>(kMaxRestart + 2)));
      attr = true;
    }
    vec::k_proj<MODE, 128><<<grid, 128, sm, st>>>(S, k, V, ldv, w, sc, lds, coef, ldc, vout, partial,
                                                   pld, out, ldo, counters);
  }
  count_launch();
  CPM_CUDA(cudaGetLastError());
  return CPM_OK;
}
}  // namespace

int launch_mdot(const vec::Seg& S, int k, const double* V, int64_t ldv, const double* w,
                const double* sc, int lds, double* partial, double* out, int ldo,
                unsigned* counters, cudaStream_t st) {
  return launch_proj<0>(S, k, V, ldv, const_cast<double*>(w), sc, lds, nullptr, 0, nullptr, partial,
                        kMaxRestart + 8, out, ldo, counters, st);
}

int launch_cgs_final(const vec::Seg& S, int k, const double* V, int64_t ldv, const double* w,
                     const double* sc, int lds, const double* coef, int ldo, double* vout,
                     double* partial, double* out, int ldn, unsigned* counters, cudaStream_t st) {
  return launch_proj<2>(S, k, V, ldv, const_cast<double*>(w), sc, lds, coef, ldo, vout, partial, 1,
                        out, ldn, counters, st);
}

int launch_cgs_update(const vec::Seg& S, int k, const double* V, int64_t ldv, double* w,
                      const double* sc, int lds, const double* coef, double* partial, double* out,
                      int ldo, unsigned* counters, cudaStream_t st) {
  return launch_proj<1>(S, k, V, ldv, w, sc, lds, coef, ldo, nullptr, partial, kMaxRestart + 8, out,
                        ldo, counters, st);
}

namespace {
constexpr int kLdc = kMaxRestart + 2;  // stride of GState::coef / red halves
constexpr int kHostCheck = 8;          // DCGS2 steps queued between host looks at st->done
// unpreconditioned GMRES uses delayed CGS2 (2 passes per step); CPM_CGS2=1 forces
// the 3-pass CGS2 of the flexible path (A/B measurements)
const bool g_force_cgs2 = [] {
  const char* v = getenv("CPM_CGS2");
  return v && *v && *v != '0';
}();
}  // namespace

int launch_dcgs_dots(const vec::Seg& S, int k, const double* V, int64_t ldv, const double* z,
                     double* partial, int pld, double* out, int ldo, unsigned* counters,
                     cudaStream_t st, const int* skip) {
  return launch_dcgs_dots_epi(S, k, V, ldv, z, partial, pld, out, ldo, counters, st, skip, vec::NoEpi());
}

int launch_dcgs_update(const vec::Seg& S, int k, double* V, int64_t ldv, const double* z,
                       const double* coef, int ldc, int64_t cstride, cudaStream_t st,
                       const int* skip) {
  const int grid = S.nseg * S.gps;
  static const bool reg = [] {
    const char* v = getenv("CPM_UPD_REG");
    return !v || *v != '0';
  }();
  if (reg && k - 1 <= 8) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_update_reg<256, 8>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z, coef,
                        ldc, cstride, skip));
  } else if (reg && k - 1 <= 16) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_update_reg<256, 16>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z, coef,
                        ldc, cstride, skip));
  } else if (reg && k - 1 <= 24) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_update_reg<256, 24>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z, coef,
                        ldc, cstride, skip));
  } else if (reg && k - 1 <= 32) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_update_reg<256, 32>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z, coef,
                        ldc, cstride, skip));
  } else if (reg && k - 1 <= 40) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_update_reg<256, 40>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z, coef,
                        ldc, cstride, skip));
  } else if (reg && k - 1 <= 52) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_update_reg<256, 52>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z, coef,
                        ldc, cstride, skip));
  } else if (reg && k - 1 <= 64) {  // one block per SM, up to 64 loads in flight per thread
    CPM_CUDA(launch_pdl(vec::k_dcgs_update_reg<256, 64, 1>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z,
                        coef, ldc, cstride, skip));
  } else if (k <= 52) {  // CPM_UPD_REG=0 (A/B)
    const size_t sm = ((size_t)k * (256 + 4) + 2 * (size_t)k) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      CPM_CUDA(cudaFuncSetAttribute(vec::k_dcgs_update<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(((size_t)64 * 260 + 128) * sizeof(double))));
      attr = true;
    }
    vec::k_dcgs_update<256><<<grid, 256, sm, st>>>(S, k, V, ldv, z, coef, ldc, cstride, skip);
  } else {  // 128-element tiles: two blocks per SM still fit (results do not depend on the tile)
    const size_t sm = ((size_t)k * (128 + 4) + 2 * (size_t)k) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      CPM_CUDA(cudaFuncSetAttribute(vec::k_dcgs_update<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(((size_t)(kMaxRestart + 1) * 132 + 2 * (kMaxRestart + 1)) * sizeof(double))));
      attr = true;
    }
    vec::k_dcgs_update<128><<<grid, 128, sm, st>>>(S, k, V, ldv, z, coef, ldc, cstride, skip);
  }
  count_launch();
  CPM_CUDA(cudaGetLastError());
  return CPM_OK;
}

namespace {

// ---------------------------------------------------------------- scalar kernels (1 thread)
__global__ void k_cycle_init(GState* st) {
  const double beta = sqrt(st->beta2);
  st->beta = beta;
  st->g[0] = beta;
  for (int i = 1; i <= kMaxRestart; ++i) st->g[i] = 0.0;
  st->sc[0] = beta > 0.0 ? 1.0 / beta : 0.0;
  st->k = 0;
  st->breakdown = 0;
  st->est = beta;
  st->done = beta <= st->target ? 1 : 0;
}

// Hessenberg column j from h1 + h2 and ||w||, Givens rotations, convergence.
__global__ void k_arnoldi_step(GState* st, int j, int m) {
  const int ld = kMaxRestart + 1;
  double* H = st->H + (size_t)j * ld;
  for (int i = 0; i <= j; ++i) H[i] = st->h1[i] + st->h2[i];
  const double nrm = sqrt(st->nrm2);
  H[j + 1] = nrm;
  for (int i = 0; i < j; ++i) {
    const double t = st->cs[i] * H[i] + st->sn[i] * H[i + 1];
    H[i + 1] = -st->sn[i] * H[i] + st->cs[i] * H[i + 1];
    H[i] = t;
  }
  const double den = hypot(H[j], H[j + 1]);
  const int brk = (H[j + 1] == 0.0) ? 1 : 0;
  if (den == 0.0) {
    st->cs[j] = 1.0;
    st->sn[j] = 0.0;
  } else {
    st->cs[j] = H[j] / den;
    st->sn[j] = H[j + 1] / den;
  }
  H[j] = st->cs[j] * H[j] + st->sn[j] * H[j + 1];
  H[j + 1] = 0.0;
  st->g[j + 1] = -st->sn[j] * st->g[j];
  st->g[j] = st->cs[j] * st->g[j];
  st->est = fabs(st->g[j + 1]);
  st->k = j + 1;
  st->its += 1;
  st->sc[j + 1] = nrm > 0.0 ? 1.0 / nrm : 0.0;
  st->breakdown = brk;
  if (st->est <= st->target || brk || j + 1 == m) st->done = 1;
}

// Delayed CGS2 step j (one thread).  Inputs (st->red, from k_dcgs_dots over the
// columns Q_0..Q_{j-1}, u_j and the vectors u_j, z = A u_j):
//   b = Q^T u_j, alpha = u_j.u_j, d = Q^T z, gamma = u_j.z.
// u_j = rho q_j + Q b with rho^2 = alpha - |b|^2 (Pythagoras), so the pending
// Hessenberg column j-1 is [cpend + b; rho] (finalised here: Givens, residual
// estimate, convergence), and A q_j = (z - Q_{<=j} g)/rho with g = Hr b, so the
// first projection of A q_j is cpend = ([d; rho mu] - g)/rho, mu = (gamma - b.d)/rho^2,
// and the next lagged vector u_{j+1} = (z - mu u_j - Q (d - mu b))/rho
// (k_dcgs_update, coefficients in st->coef).
constexpr int kStepThreads = 128;
// Run by one block of nt = blockDim.x threads (<= 256): the k_dcgs_step kernel, or
// the block of k_dcgs_dots that finishes the reduction (single-GPU solves, where
// no allreduce sits between the two).
__device__ void dcgs_step_body(GState* st, int j, int m, int maxit) {
  if (st->done) return;  // a step queued past convergence
  const int ld = kMaxRestart + 1, k = j + 1, tid = threadIdx.x, nt = blockDim.x;
  const double* b = st->red;
  const double* d = st->red + k;
  __shared__ double sbb[8], sbd[8];
  __shared__ int sdone;
  double pbb = 0.0, pbd = 0.0;
  for (int i = tid; i < j; i += nt) {
    pbb += b[i] * b[i];
    pbd += b[i] * d[i];
  }
  pbb = vec::warp_sum(pbb);
  pbd = vec::warp_sum(pbd);
  if ((tid & 31) == 0) {
    sbb[tid >> 5] = pbb;
    sbd[tid >> 5] = pbd;
  }
  __syncthreads();
  double bb = 0.0, bd = 0.0;
  for (int w = 0; w < nt / 32; ++w) {
    bb += sbb[w];
    bd += sbd[w];
  }
  const double alpha = st->red[j], gamma = st->red[k + j];
  const double rho2 = alpha - bb;
  const int brk = !(rho2 > 1e-28 * alpha);
  const double rho = brk ? 0.0 : sqrt(rho2);
  if (j >= 1)
    for (int i = tid; i < j; i += nt) st->Hr[(size_t)(j - 1) * ld + i] = st->cpend[i] + b[i];
  __syncthreads();
  if (tid == 0) {
    sdone = 0;
    if (j == 0) {
      st->g[0] *= rho;  // u_0 = r / beta: r = (beta rho) q_0
      st->est = fabs(st->g[0]);
      if (brk) sdone = 1;
    } else {
      double* Hr = st->Hr + (size_t)(j - 1) * ld;
      double* H = st->H + (size_t)(j - 1) * ld;
      Hr[j] = rho;
      for (int i = 0; i <= j; ++i) H[i] = Hr[i];
      const int c = j - 1;  // column index
      for (int i = 0; i < c; ++i) {
        const double t = st->cs[i] * H[i] + st->sn[i] * H[i + 1];
        H[i + 1] = -st->sn[i] * H[i] + st->cs[i] * H[i + 1];
        H[i] = t;
      }
      const double den = hypot(H[c], H[c + 1]);
      if (den == 0.0) {
        st->cs[c] = 1.0;
        st->sn[c] = 0.0;
      } else {
        st->cs[c] = H[c] / den;
        st->sn[c] = H[c + 1] / den;
      }
      H[c] = st->cs[c] * H[c] + st->sn[c] * H[c + 1];
      H[c + 1] = 0.0;
      st->g[c + 1] = -st->sn[c] * st->g[c];
      st->g[c] = st->cs[c] * st->g[c];
      st->est = fabs(st->g[c + 1]);
      st->k = j;
      st->its += 1;
      st->breakdown = brk;
      if (st->est <= st->target || brk || j == m || st->its >= maxit) sdone = 1;
    }
    if (sdone) st->done = 1;
  }
  __syncthreads();
  if (sdone) return;
  const double mu = (gamma - bd) / rho2;
  double* cb = st->coef;
  double* ce = st->coef + (kMaxRestart + 2);
  for (int l = tid; l <= j; l += nt) {
    double gl = 0.0;  // (Hr b)_l, Hr[l, i] = 0 for l > i + 1
    for (int i = (l > 0 ? l - 1 : 0); i < j; ++i) gl += st->Hr[(size_t)i * ld + l] * b[i];
    const double ql = l < j ? d[l] : rho * mu;
    st->cpend[l] = (ql - gl) / rho;
  }
  for (int i = tid; i < j; i += nt) {
    cb[i] = b[i];
    ce[i] = d[i] - mu * b[i];
  }
  if (tid == 0) {
    st->coef[2 * (kMaxRestart + 2)] = rho;
    st->coef[2 * (kMaxRestart + 2) + 1] = mu;
  }
}
__global__ void __launch_bounds__(kStepThreads) k_dcgs_step(GState* st, int j, int m, int maxit) {
  dcgs_step_body(st, j, m, maxit);
}
struct StepEpi {
  GState* st;
  int j, m, maxit;
  __device__ void operator()(int) const { dcgs_step_body(st, j, m, maxit); }
};

// Back substitution H(0:k,0:k) y = g(0:k), one warp (lanes split the row sums).
__global__ void k_lsq(GState* st) {
  const int ld = kMaxRestart + 1;
  const int k = st->k;
  const int lane = threadIdx.x;
  for (int i = k - 1; i >= 0; --i) {
    double s = 0.0;
    for (int q = i + 1 + lane; q < k; q += 32) s += st->H[(size_t)q * ld + i] * st->y[q];
    s = vec::warp_sum(s);
    if (lane == 0) st->y[i] = (st->g[i] - s) / st->H[(size_t)i * ld + i];
    __syncwarp();
    __threadfence_block();
  }
}

}  // namespace

// ---------------------------------------------------------------- host side
int Workspace::ensure(int64_t n_, int m_, bool flex_) {
  if (n_ == n && m_ == m && flex_ == flex && V) return CPM_OK;
  release();
  n = n_;
  m = m_;
  flex = flex_;
  ldv = (n + 63) / 64 * 64;
  auto al = [&](void** p, size_t bytes) -> int {
    if (cudaMalloc(p, std::max<size_t>(bytes, 8)) != cudaSuccess)
      return fail(CPM_ERR_NOMEM, "GMRES workspace allocation failed");
    return CPM_OK;
  };
  CPM_TRY(al((void**)&V, sizeof(double) * (size_t)ldv * (m + 1)));
  if (flex) CPM_TRY(al((void**)&Z, sizeof(double) * (size_t)ldv * m));
  CPM_TRY(al((void**)&w, sizeof(double) * (size_t)ldv));
  CPM_TRY(al((void**)&t, sizeof(double) * (size_t)ldv));
  CPM_TRY(al((void**)&partial, sizeof(double) * (size_t)kMaxBlocks * (kMaxRestart + 8)));
  CPM_TRY(al((void**)&st, sizeof(GState)));
  CPM_TRY(al((void**)&segoff, sizeof(int64_t) * 2));
  CPM_CUDA(cudaMemset(st, 0, sizeof(GState)));
  int64_t off[2] = {0, n};
  CPM_CUDA(cudaMemcpy(segoff, off, sizeof(off), cudaMemcpyHostToDevice));
  const int64_t nsub = (n + vec::VB - 1) / vec::VB;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // 2 blocks per SM: each thread streams many elements; few partials to combine
  gps = (int)std::max<int64_t>(1, std::min<int64_t>(nsub, 2 * (int64_t)sms));
  if (cudaMallocHost((void**)&hst, sizeof(HostState)) != cudaSuccess)
    return fail(CPM_ERR_NOMEM, "pinned host state allocation failed");
  return CPM_OK;
}

void Workspace::release() {
  if (V) cudaFree(V);
  if (Z) cudaFree(Z);
  if (w) cudaFree(w);
  if (t) cudaFree(t);
  if (partial) cudaFree(partial);
  if (st) cudaFree(st);
  if (segoff) cudaFree(segoff);
  if (hst) cudaFreeHost(hst);
  V = Z = w = t = partial = nullptr;
  st = nullptr;
  segoff = nullptr;
  hst = nullptr;
  n = 0;
  m = 0;
}

namespace {
int fetch_state(Workspace& ws, cudaStream_t s) {
  CPM_CUDA(cudaMemcpyAsync(&ws.hst->k, &ws.st->k, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaMemcpyAsync(&ws.hst->est, &ws.st->est, sizeof(double) * 2, cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  return CPM_OK;
}
}  // namespace

int gmres_device(const LinOp& A, const PrecOp* M, const double* b, double* x, int64_t n,
                 double rtol, int m, int maxit, Workspace& ws, cpm_solve_stats* stats,
                 cudaStream_t s) {
  auto t0 = std::chrono::steady_clock::now();
  if (m < 1 || m > kMaxRestart) return fail(CPM_ERR_ARG, "cpm_solve: restart must be in [1, 128]");
  if (!(rtol > 0.0)) return fail(CPM_ERR_ARG, "cpm_solve: rtol must be > 0");
  const bool flex = M != nullptr;
  CPM_TRY(ws.ensure(n, m, flex));
  const vec::Seg S{ws.segoff, 1, ws.gps};
  const int G = ws.gps;
  GState* st = ws.st;
  unsigned* cnt = st->counter;  // address arithmetic on a device pointer

  auto allreduce = [&](double* buf, size_t nv) -> int {
    return A.allreduce ? A.allreduce(buf, nv, s) : CPM_OK;
  };
  {
    ProfScope ps(K_OTHER, s);
    vec::k_sub_nrm2<<<G, VB, 0, s>>>(S, b, nullptr, nullptr, ws.partial, &st->beta2, 0, cnt);
    count_launch();
  }
  CPM_TRY(allreduce(&st->beta2, 1));
  CPM_CUDA(cudaMemcpyAsync(&ws.hst->est, &st->beta2, sizeof(double), cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  const double bnorm = sqrt(ws.hst->est);
  if (!std::isfinite(bnorm)) return fail(CPM_ERR_ARG, "cpm_solve: right-hand side is not finite");
  const double target = rtol * bnorm;
  CPM_CUDA(cudaMemcpyAsync(&st->target, &target, sizeof(double), cudaMemcpyHostToDevice, s));
  CPM_CUDA(cudaMemsetAsync(&st->its, 0, sizeof(int), s));

  int its = 0, cycles = 0, converged = 0, breakdown = 0;
  double est = 0.0;
  if (bnorm == 0.0) {
    CPM_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    converged = 1;
  }
  while (!converged) {
    // r = b - A x  -> V_0 ; beta
    CPM_TRY(A.apply(x, ws.t, nullptr, nullptr, s));
    {
      ProfScope ps(K_AXPY, s);
      vec::k_sub_nrm2<<<G, VB, 0, s>>>(S, b, ws.t, ws.V, ws.partial, &st->beta2, 0, cnt);
      count_launch();
      CPM_TRY(allreduce(&st->beta2, 1));
      k_cycle_init<<<1, 1, 0, s>>>(st);
      count_launch();
    }
    CPM_TRY(fetch_state(ws, s));
    if (ws.hst->done) {  // beta <= target
      converged = 1;
      est = ws.hst->est;
      break;
    }
    if (its >= maxit) break;
    ++cycles;
    const int its_cycle0 = its;
    if (!flex && !g_force_cgs2) {
      // delayed CGS2: V_0 = r / beta is the first lagged vector
      {
        ProfScope ps(K_AXPY, s);
        vec::k_scale<<<G, VB, 0, s>>>(S, ws.V, st->sc, 0, 0, ws.V);
        count_launch();
      }
      // Steps are queued without a host round trip; st->done (set by the step
      // kernel at convergence, breakdown, the end of the cycle or maxit) turns the
      // kernels of steps queued past it into no-ops.  The host looks every
      // kHostCheck steps only to stop queueing.
      const int* skip = &st->done;
      for (int j = 0; j <= m; ++j) {
        double* Vj = ws.V + (size_t)j * ws.ldv;
        if (j < m) CPM_TRY(A.apply(Vj, ws.w, nullptr, skip, s));  // z = A u_j
        const int k = j + 1;
        if (!A.allreduce) {  // one GPU: the reducing block runs the step (no extra launch)
          ProfScope ps(K_MDOT, s);
          CPM_TRY(launch_dcgs_dots_epi(S, k, ws.V, ws.ldv, ws.w, ws.partial, 2 * kLdc + 8, st->red, 0,
                                       cnt + 1, s, skip, StepEpi{st, j, m, maxit}));
        } else {
          {
            ProfScope ps(K_MDOT, s);
            CPM_TRY(launch_dcgs_dots(S, k, ws.V, ws.ldv, ws.w, ws.partial, 2 * kLdc + 8, st->red, 0,
                                     cnt + 1, s, skip));
            CPM_TRY(allreduce(st->red, 2 * k));
          }
          ProfScope ps(K_OTHER, s);
          k_dcgs_step<<<1, kStepThreads, 0, s>>>(st, j, m, maxit);
          count_launch();
        }
        if (j < m) {
          ProfScope ps(K_CGS_UPDATE, s);
          CPM_TRY(launch_dcgs_update(S, k, ws.V, ws.ldv, ws.w, st->coef, kLdc, 0, s, skip));
        }
        if ((j + 1) % kHostCheck == 0 || j == m) {
          CPM_TRY(fetch_state(ws, s));
          its = ws.hst->its;
          if (ws.hst->done) break;
        }
      }
    } else
    for (int j = 0; j < m; ++j) {
      double* Vj = ws.V + (size_t)j * ws.ldv;
      if (flex) {
        {
          ProfScope ps(K_AXPY, s);
          vec::k_scale<<<G, VB, 0, s>>>(S, Vj, st->sc, 0, j, ws.w);
          count_launch();
        }
        double* Zj = ws.Z + (size_t)j * ws.ldv;
        CPM_TRY(M->apply(ws.w, Zj, s));
        CPM_TRY(A.apply(Zj, ws.w, nullptr, nullptr, s));
      } else {
        CPM_TRY(A.apply(Vj, ws.w, &st->sc[j], nullptr, s));
      }
      const int k = j + 1;
      {
        ProfScope ps(K_MDOT, s);
        CPM_TRY(launch_mdot(S, k, ws.V, ws.ldv, ws.w, st->sc, 0, ws.partial, st->h1, 0, cnt + 1, s));
        CPM_TRY(allreduce(st->h1, k));
      }
      {
        ProfScope ps(K_CGS_UPDATE, s);
        CPM_TRY(launch_cgs_update(S, k, ws.V, ws.ldv, ws.w, st->sc, 0, st->h1, ws.partial, st->h2, 0,
                                  cnt + 2, s));
        CPM_TRY(allreduce(st->h2, k));
      }
      {
        ProfScope ps(K_CGS_FINAL, s);
        CPM_TRY(launch_cgs_final(S, k, ws.V, ws.ldv, ws.w, st->sc, 0, st->h2, 0,
                                 ws.V + (size_t)(j + 1) * ws.ldv, ws.partial, &st->nrm2, 0, cnt + 3,
                                 s));
        CPM_TRY(allreduce(&st->nrm2, 1));
      }
      {
        ProfScope ps(K_OTHER, s);
        k_arnoldi_step<<<1, 1, 0, s>>>(st, j, m);
        count_launch();
      }
      CPM_TRY(fetch_state(ws, s));
      its = ws.hst->its;
      if (ws.hst->done || its >= maxit) break;
    }
    {
      ProfScope ps(K_AXPY, s);
      k_lsq<<<1, 32, 0, s>>>(st);
      count_launch();
      const bool scaled = !flex && g_force_cgs2;  // CGS2 keeps the basis unnormalised
      vec::k_combine<<<G, VB, 0, s>>>(S, flex ? ws.Z : ws.V, ws.ldv, st->y, 0, scaled ? st->sc : nullptr, 0,
                                      &st->k, 0, 0, nullptr, nullptr, nullptr, x, 1);
      count_launch();
    }
    CPM_CUDA(cudaGetLastError());
    CPM_TRY(fetch_state(ws, s));
    est = ws.hst->est;
    breakdown = ws.hst->breakdown;
    its = ws.hst->its;
    if (est <= target) {
      converged = 1;
      break;
    }
    if (its >= maxit) break;
    // no Arnoldi step completed (a breakdown at j = 0: a non-finite x0 or residual)
    // or a non-finite estimate: restarting cannot make progress, stop and report it
    if (its == its_cycle0 || !std::isfinite(est)) {
      breakdown = 1;
      break;
    }
  }
  double rtrue = 0.0;
  if (stats) {
    CPM_TRY(A.apply(x, ws.t, nullptr, nullptr, s));
    {
      ProfScope ps(K_OTHER, s);
      vec::k_sub_nrm2<<<G, VB, 0, s>>>(S, b, ws.t, nullptr, ws.partial, &st->beta2, 0, cnt);
      count_launch();
    }
    CPM_TRY(allreduce(&st->beta2, 1));
    CPM_CUDA(cudaMemcpyAsync(&ws.hst->est, &st->beta2, sizeof(double), cudaMemcpyDeviceToHost, s));
    CPM_CUDA(cudaStreamSynchronize(s));
    rtrue = sqrt(ws.hst->est);
    stats->iterations = its;
    stats->converged = converged;
    stats->cycles = cycles;
    stats->breakdown = breakdown;
    stats->resid_est = est;
    stats->resid_true = rtrue;
    stats->bnorm = bnorm;
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  CPM_CUDA(cudaStreamSynchronize(s));
  return CPM_OK;
}

}  // namespace cpm
