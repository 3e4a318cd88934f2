// krylov.cu — restarted (F)GMRES(m) with CGS2 Arnoldi (north_star item 3).
//
// Textbook GMRES (Saad, Alg. 6.9/6.11) with classical Gram-Schmidt applied
// twice; conventions of reading R5 (shared with oracle/krylov.py): x0 from the
// caller, convergence when the Givens estimate |g_{j+1}| <= rtol ||b||, the
// iteration count is the number of Arnoldi steps, right preconditioning in the
// flexible form (Z_j = M v_j stored).
//
// Device-resident design:
//  * The basis is stored UNNORMALISED, V_i = w_i, with sc_i = 1/||w_i|| kept
//    on the device; every kernel applies sc_i on the fly, so no normalisation
//    pass exists (one HBM pass per Arnoldi step saved).
//  * One Arnoldi step = apply (2 kernels) + 3 fused passes over the basis:
//      mdot        h1 = V^T w
//      cgs_update  w <- w - V h1  AND  h2 = V^T w   (same sweep, sub-chunk in smem)
//      cgs_final   V_{j+1} <- w - V h2  AND  ||V_{j+1}||^2
//    followed by a one-thread Hessenberg/Givens kernel.  Reductions are
//    deterministic: per-block partials in a fixed sub-chunk assignment, summed
//    in block order by the last block to finish (threadfence + counter).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include "internal.cuh"
#include "krylov.cuh"

namespace cpm {
namespace {

constexpr int VB = 256;                 // threads per block, vector kernels
constexpr int SUB = 256;                // elements per sub-chunk
constexpr int NQ = (kMaxRestart + 1 + 7) / 8;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-sum of one value per thread (deterministic order).
__device__ double block_sum(double v) {
  __shared__ double sw[VB / 32];
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sw[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = lane < VB / 32 ? sw[lane] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// Last block: out[i] = scale_i * sum_b partial[b * k + i], i < k.
__device__ void last_block_finish(const double* partial, int k, const double* sc, double* out,
                                  unsigned* counter) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = warp; i < k; i += VB / 32) {
    double a = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) a += __ldcg(partial + (size_t)b * k + i);
    a = warp_sum(a);
    if (lane == 0) out[i] = sc ? a * sc[i] : a;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// ---------------------------------------------------------------- mdot: out_i = sc_i <V_i, w>
__global__ void __launch_bounds__(VB) k_mdot(int64_t n, int k, const double* __restrict__ V,
                                             int64_t ldv, const double* __restrict__ w,
                                             const double* __restrict__ sc, double* partial,
                                             double* out, unsigned* counter) {
  __shared__ double ws[SUB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  const int64_t nsub = (n + SUB - 1) / SUB;
  for (int64_t s = blockIdx.x; s < nsub; s += gridDim.x) {
    const int64_t base = s * SUB;
    const int64_t e = base + threadIdx.x;
    ws[threadIdx.x] = e < n ? __ldg(w + e) : 0.0;
    __syncthreads();
    const int lim = (int)((n - base) < SUB ? (n - base) : SUB);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = warp + 8 * q;
      if (i < k) {
        const double* vi = V + (size_t)i * ldv + base;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int r = 0; r < SUB / 32; r += 2) {
          const int l0 = lane + 32 * r, l1 = l0 + 32;
          if (l0 < lim) a0 += __ldg(vi + l0) * ws[l0];
          if (l1 < lim) a1 += __ldg(vi + l1) * ws[l1];
        }
        acc[q] += a0 + a1;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int i = warp + 8 * q;
    if (i < k) {
      const double v = warp_sum(acc[q]);
      if (lane == 0) partial[(size_t)blockIdx.x * k + i] = v;
    }
  }
  last_block_finish(partial, k, sc, out, counter);
}

// ---------------------------------------------------------------- cgs_update
// w <- w - sum_i coef_i sc_i V_i   and   out_i = sc_i <V_i, w_new>.
__global__ void __launch_bounds__(VB) k_cgs_update(int64_t n, int k, const double* __restrict__ V,
                                                   int64_t ldv, double* __restrict__ w,
                                                   const double* __restrict__ sc,
                                                   const double* __restrict__ coef,
                                                   double* partial, double* out,
                                                   unsigned* counter) {
  __shared__ double ws[SUB];
  __shared__ double cf[kMaxRestart + 1];
  for (int i = threadIdx.x; i < k; i += VB) cf[i] = coef[i] * sc[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  const int64_t nsub = (n + SUB - 1) / SUB;
  for (int64_t s = blockIdx.x; s < nsub; s += gridDim.x) {
    const int64_t base = s * SUB;
    const int64_t e = base + threadIdx.x;
    double v = 0.0;
    if (e < n) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int i = 0;
      for (; i + 3 < k; i += 4) {
        s0 += cf[i] * __ldg(V + (size_t)i * ldv + e);
        s1 += cf[i + 1] * __ldg(V + (size_t)(i + 1) * ldv + e);
        s2 += cf[i + 2] * __ldg(V + (size_t)(i + 2) * ldv + e);
        s3 += cf[i + 3] * __ldg(V + (size_t)(i + 3) * ldv + e);
      }
      for (; i < k; ++i) s0 += cf[i] * __ldg(V + (size_t)i * ldv + e);
      v = w[e] - ((s0 + s1) + (s2 + s3));
      w[e] = v;
    }
    ws[threadIdx.x] = v;
    __syncthreads();
    const int lim = (int)((n - base) < SUB ? (n - base) : SUB);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = warp + 8 * q;
      if (i < k) {
        const double* vi = V + (size_t)i * ldv + base;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int r = 0; r < SUB / 32; r += 2) {
          const int l0 = lane + 32 * r, l1 = l0 + 32;
          if (l0 < lim) a0 += __ldg(vi + l0) * ws[l0];
          if (l1 < lim) a1 += __ldg(vi + l1) * ws[l1];
        }
        acc[q] += a0 + a1;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int i = warp + 8 * q;
    if (i < k) {
      const double v = warp_sum(acc[q]);
      if (lane == 0) partial[(size_t)blockIdx.x * k + i] = v;
    }
  }
  last_block_finish(partial, k, sc, out, counter);
}

// ---------------------------------------------------------------- cgs_final
// vout <- w - sum_i coef_i sc_i V_i ;  out = ||vout||^2.  (vout may alias w)
__global__ void __launch_bounds__(VB) k_cgs_final(int64_t n, int k, const double* __restrict__ V,
                                                  int64_t ldv, const double* w,
                                                  const double* __restrict__ sc,
                                                  const double* __restrict__ coef, double* vout,
                                                  double* partial, double* out,
                                                  unsigned* counter) {
  __shared__ double cf[kMaxRestart + 1];
  for (int i = threadIdx.x; i < k; i += VB) cf[i] = coef ? coef[i] * sc[i] : 0.0;
  __syncthreads();
  double acc = 0.0;
  const int64_t nsub = (n + SUB - 1) / SUB;
  for (int64_t s = blockIdx.x; s < nsub; s += gridDim.x) {
    const int64_t e = s * SUB + threadIdx.x;
    if (e < n) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int i = 0;
      for (; i + 3 < k; i += 4) {
        s0 += cf[i] * __ldg(V + (size_t)i * ldv + e);
        s1 += cf[i + 1] * __ldg(V + (size_t)(i + 1) * ldv + e);
        s2 += cf[i + 2] * __ldg(V + (size_t)(i + 2) * ldv + e);
        s3 += cf[i + 3] * __ldg(V + (size_t)(i + 3) * ldv + e);
      }
      for (; i < k; ++i) s0 += cf[i] * __ldg(V + (size_t)i * ldv + e);
      const double v = w[e] - ((s0 + s1) + (s2 + s3));
      vout[e] = v;
      acc += v * v;
    }
  }
  const double b = block_sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = b;
  last_block_finish(partial, 1, nullptr, out, counter);
}

// ---------------------------------------------------------------- misc vector kernels
// out = b - t  (into out), partial ||out||^2 -> res
__global__ void __launch_bounds__(VB) k_sub_nrm2(int64_t n, const double* __restrict__ b,
                                                 const double* __restrict__ t, double* out,
                                                 double* partial, double* res,
                                                 unsigned* counter) {
  double acc = 0.0;
  const int64_t nsub = (n + SUB - 1) / SUB;
  for (int64_t s = blockIdx.x; s < nsub; s += gridDim.x) {
    const int64_t e = s * SUB + threadIdx.x;
    if (e < n) {
      const double v = b[e] - (t ? t[e] : 0.0);
      if (out) out[e] = v;
      acc += v * v;
    }
  }
  const double bs = block_sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = bs;
  last_block_finish(partial, 1, nullptr, res, counter);
}

// x += sum_{i<k} y_i * (sc ? sc_i : 1) * V_i
__global__ void __launch_bounds__(VB) k_update_x(int64_t n, const GState* st,
                                                 const double* __restrict__ V, int64_t ldv,
                                                 bool use_sc, double* __restrict__ x) {
  __shared__ double cf[kMaxRestart + 1];
  const int k = st->k;
  for (int i = threadIdx.x; i < k; i += VB) cf[i] = st->y[i] * (use_sc ? st->sc[i] : 1.0);
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)VB + threadIdx.x; e < n; e += (int64_t)gridDim.x * VB) {
    double s0 = 0.0;
    for (int i = 0; i < k; ++i) s0 += cf[i] * __ldg(V + (size_t)i * ldv + e);
    x[e] += s0;
  }
}

// y_i <- scale * x_i
__global__ void k_scale(int64_t n, const double* __restrict__ x, const double* __restrict__ sc,
                        double* __restrict__ y) {
  const double s = *sc;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    y[e] = s * x[e];
}

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

// Back substitution H(0:k,0:k) y = g(0:k).
__global__ void k_lsq(GState* st) {
  const int ld = kMaxRestart + 1;
  const int k = st->k;
  for (int i = k - 1; i >= 0; --i) {
    double s = st->g[i];
    for (int q = i + 1; q < k; ++q) s -= st->H[(size_t)q * ld + i] * st->y[q];
    st->y[i] = s / st->H[(size_t)i * ld + i];
  }
}

inline int vgrid(int64_t n) {
  const int64_t nsub = (n + SUB - 1) / SUB;
  return (int)std::max<int64_t>(1, std::min<int64_t>(nsub, 148 * 8));
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
  CPM_TRY(al((void**)&partial, sizeof(double) * (size_t)148 * 8 * (kMaxRestart + 1)));
  CPM_TRY(al((void**)&st, sizeof(GState)));
  CPM_CUDA(cudaMemset(st, 0, sizeof(GState)));
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
  if (hst) cudaFreeHost(hst);
  V = Z = w = t = partial = nullptr;
  st = nullptr;
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
  const int G = vgrid(n);
  GState* st = ws.st;
  unsigned* cnt = st->counter;  // device address arithmetic on a device pointer

  // ||b||, target
  {
    ProfScope ps(K_OTHER, s);
    k_sub_nrm2<<<G, VB, 0, s>>>(n, b, nullptr, nullptr, ws.partial, &st->beta2, cnt);
    count_launch();
  }
  CPM_CUDA(cudaMemcpyAsync(&ws.hst->est, &st->beta2, sizeof(double), cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  const double bnorm = sqrt(ws.hst->est);
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
    CPM_TRY(A.apply(x, ws.t, nullptr, s));
    {
      ProfScope ps(K_AXPY, s);
      k_sub_nrm2<<<G, VB, 0, s>>>(n, b, ws.t, ws.V, ws.partial, &st->beta2, cnt);
      count_launch();
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
    for (int j = 0; j < m; ++j) {
      double* Vj = ws.V + (size_t)j * ws.ldv;
      if (flex) {
        {
          ProfScope ps(K_AXPY, s);
          k_scale<<<G, VB, 0, s>>>(n, Vj, &st->sc[j], ws.w);
          count_launch();
        }
        double* Zj = ws.Z + (size_t)j * ws.ldv;
        CPM_TRY(M->apply(ws.w, Zj, s));
        CPM_TRY(A.apply(Zj, ws.w, nullptr, s));
      } else {
        CPM_TRY(A.apply(Vj, ws.w, &st->sc[j], s));
      }
      const int k = j + 1;
      {
        ProfScope ps(K_MDOT, s);
        k_mdot<<<G, VB, 0, s>>>(n, k, ws.V, ws.ldv, ws.w, st->sc, ws.partial, st->h1, cnt + 1);
        count_launch();
      }
      {
        ProfScope ps(K_CGS_UPDATE, s);
        k_cgs_update<<<G, VB, 0, s>>>(n, k, ws.V, ws.ldv, ws.w, st->sc, st->h1, ws.partial,
                                      st->h2, cnt + 2);
        count_launch();
      }
      {
        ProfScope ps(K_CGS_FINAL, s);
        k_cgs_final<<<G, VB, 0, s>>>(n, k, ws.V, ws.ldv, ws.w, st->sc, st->h2,
                                     ws.V + (size_t)(j + 1) * ws.ldv, ws.partial, &st->nrm2,
                                     cnt + 3);
        count_launch();
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
      k_lsq<<<1, 1, 0, s>>>(st);
      count_launch();
      k_update_x<<<G, VB, 0, s>>>(n, st, flex ? ws.Z : ws.V, ws.ldv, !flex, x);
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
  }
  // true residual
  double rtrue = 0.0;
  if (stats) {
    CPM_TRY(A.apply(x, ws.t, nullptr, s));
    {
      ProfScope ps(K_OTHER, s);
      k_sub_nrm2<<<G, VB, 0, s>>>(n, b, ws.t, nullptr, ws.partial, &st->beta2, cnt);
      count_launch();
    }
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
    stats->seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  CPM_CUDA(cudaStreamSynchronize(s));
  return CPM_OK;
}

// Exposed helpers for the RAS local solver / tests.
int vec_nrm2(const double* x, int64_t n, double* d_out, Workspace& ws, cudaStream_t s) {
  const int G = vgrid(n);
  k_sub_nrm2<<<G, VB, 0, s>>>(n, x, nullptr, nullptr, ws.partial, d_out, ws.st->counter);
  count_launch();
  CPM_CUDA(cudaGetLastError());
  return CPM_OK;
}

}  // namespace cpm
