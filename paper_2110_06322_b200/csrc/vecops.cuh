// vecops.cuh — segmented, deterministic Krylov vector kernels (private).
//
// A "segmented" vector is the concatenation of nseg independent vectors
// (segment s = elements [off[s], off[s+1])).  The global GMRES uses one segment;
// the RAS preconditioner runs all subdomain GMRES solves as segments of one
// batched vector.  Grid = nseg * gps blocks; block b works on segment b / gps and
// visits the segment's elements lb*VB + t, lb*VB + t + gps*VB, ... (lb = b % gps),
// so every reduction has a fixed association order: per-thread accumulation in
// element order, warp shuffle tree, warps in index order, blocks in index order
// (summed by the last block of the segment to finish; threadfence + counter).
//
// Basis vectors V_i are stored unnormalised; sc[s*lds + i] = 1/||V_i|| of
// segment s is applied on the fly.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "internal.cuh"

namespace cpm {
namespace vec {

constexpr int VB = 256;

struct Seg {
  const int64_t* off;  // device, nseg + 1
  int nseg;
  int gps;             // blocks per segment
  int aligned = 0;     // host hint: every off[s] is even (16-byte aligned segment starts)
};

__device__ __forceinline__ void cp_commit_v() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all_v() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum partial[(base + b) * pld + i] over b < gps, lane-strided with 4 independent
// accumulators (loads in flight), then across the warp.  Fixed order.
__device__ __forceinline__ double partial_sum(const double* partial, size_t base, int pld, int gps,
                                              int i, int lane) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int b = lane;
  for (; b + 96 < gps; b += 128) {
    a0 += __ldcg(partial + (base + b) * pld + i);
    a1 += __ldcg(partial + (base + b + 32) * pld + i);
    a2 += __ldcg(partial + (base + b + 64) * pld + i);
    a3 += __ldcg(partial + (base + b + 96) * pld + i);
  }
  for (; b < gps; b += 32) a0 += __ldcg(partial + (base + b) * pld + i);
  return warp_sum((a0 + a1) + (a2 + a3));
}

// partial_sum of two columns i, i2 at once (loads of both in flight); per column
// the same order as partial_sum.
__device__ __forceinline__ void partial_sum2(const double* partial, size_t base, int pld, int gps,
                                             int i, int i2, int lane, double& r, double& r2) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  int b = lane;
  for (; b + 96 < gps; b += 128) {
    const double* p = partial + (base + b) * pld;
    a0 += __ldcg(p + i);
    c0 += __ldcg(p + i2);
    a1 += __ldcg(p + 32 * (size_t)pld + i);
    c1 += __ldcg(p + 32 * (size_t)pld + i2);
    a2 += __ldcg(p + 64 * (size_t)pld + i);
    c2 += __ldcg(p + 64 * (size_t)pld + i2);
    a3 += __ldcg(p + 96 * (size_t)pld + i);
    c3 += __ldcg(p + 96 * (size_t)pld + i2);
  }
  for (; b < gps; b += 32) {
    a0 += __ldcg(partial + (base + b) * pld + i);
    c0 += __ldcg(partial + (base + b) * pld + i2);
  }
  r = warp_sum((a0 + a1) + (a2 + a3));
  r2 = warp_sum((c0 + c1) + (c2 + c3));
}

// Reduce acc[0..k) over the block into partial[blockIdx.x * pld + i]; then the
// last block of the segment writes out[s*ldo + i] = scale_i * sum_b partial.
template <int KMAX>
__device__ __forceinline__ void block_then_segment_reduce(const double (&acc)[KMAX], int k,
                                                          double* partial, int pld, int s,
                                                          int gps, const double* sc, int lds,
                                                          double* out, int ldo,
                                                          unsigned* counters) {
  __shared__ double red[VB / 32][KMAX];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    if (i < k) {
      const double v = warp_sum(acc[i]);
      if (lane == 0) red[warp][i] = v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += VB) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < VB / 32; ++w) t += red[w][i];
    partial[(size_t)blockIdx.x * pld + i] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counters + s, 1u) == (unsigned)gps - 1u);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = warp; i < k; i += VB / 32) {
    const double a = partial_sum(partial, (size_t)s * gps, pld, gps, i, lane);
    if (lane == 0) out[(size_t)s * ldo + i] = sc ? a * sc[(size_t)s * lds + i] : a;
  }
  if (threadIdx.x == 0) counters[s] = 0u;
}

// out_i = sc_i <V_i, w>  (per segment).  Vectors in groups of 8: per group each
// thread streams its elements with 8 independent loads per element (w re-read
// from L1/L2 per group), so only 8 accumulators live in registers and
// occupancy stays high; one block reduction per group.
static __global__ void __launch_bounds__(VB) k_mdot8(Seg S, int k, const double* __restrict__ V,
                                              int64_t ldv, const double* __restrict__ w,
                                              const double* __restrict__ sc, int lds,
                                              double* partial, int pld, double* out, int ldo,
                                              unsigned* counters) {
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  __shared__ double red[VB / 32][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int g = 0; g < k; g += 8) {
    const int kg = k - g < 8 ? k - g : 8;
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    const double* Vg = V + (size_t)g * ldv + o0;
    for (int64_t e = (int64_t)lb * VB + threadIdx.x; e < n; e += (int64_t)S.gps * VB) {
      const double wv = __ldg(w + o0 + e);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < kg) acc[q] += __ldcs(Vg + (size_t)q * ldv + e) * wv;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double v = warp_sum(acc[q]);
      if (lane == 0) red[warp][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < kg) {
      double t = 0.0;
#pragma unroll
      for (int ww = 0; ww < VB / 32; ++ww) t += red[ww][threadIdx.x];
      partial[(size_t)blockIdx.x * pld + g + threadIdx.x] = t;
    }
    __syncthreads();
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counters + s, 1u) == (unsigned)S.gps - 1u);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = warp; i < k; i += VB / 32) {
    const double a = partial_sum(partial, (size_t)s * S.gps, pld, S.gps, i, lane);
    if (lane == 0) out[(size_t)s * ldo + i] = sc ? a * sc[(size_t)s * lds + i] : a;
  }
  if (threadIdx.x == 0) counters[s] = 0u;
}

// ---------------------------------------------------------------- tile projections
// One kernel per pass over the basis, MODE:
//   0 (mdot)    out_i = sc_i <V_i, w>
//   1 (update)  w <- w - sum_i cf_i V_i,  out_i = sc_i <V_i, w_new>      (cf_i = coef_i sc_i)
//   2 (final)   vout <- w - sum_i cf_i V_i,  out_0 = ||vout||^2
// A block of TB threads streams tiles of TB consecutive elements of its segment
// (tiles lb, lb + gps, ... : fixed order).  Per tile every thread cp.async-copies
// its element of V_0 .. V_{k-1} into shared memory (k independent 8-byte copies
// in flight per thread: the pass runs at HBM bandwidth), forms its w value, and
// for the dots the threads, grouped P per column, reduce the tile's column
// products from shared memory.  V is read from HBM exactly once per pass.
__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(gmem));
}

template <int MODE, int TB>
static __global__ void __launch_bounds__(TB) k_proj(Seg S, int k, const double* __restrict__ V,
                                                    int64_t ldv, double* w,
                                                    const double* __restrict__ sc, int lds,
                                                    const double* __restrict__ coef, int ldc,
                                                    double* vout, double* partial, int pld,
                                                    double* out, int ldo, unsigned* counters) {
  constexpr int SV = TB + 4;  // padded column stride (bank spread of the column dots)
  extern __shared__ double smp[];
  double* sv = smp;            // k columns of SV
  double* sw = sv + (size_t)k * SV;
  double* cf = sw + TB;        // k
  double* cs = cf + k;         // TB / 32 warp sums (MODE 2)
  __shared__ bool last;
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (MODE != 0)
    for (int i = tid; i < k; i += TB) cf[i] = coef[(size_t)s * ldc + i] * sc[(size_t)s * lds + i];
  int kp = 8;
  while (kp < k) kp <<= 1;
  const int P = kp >= TB ? 1 : TB / kp;  // threads per column (<= 32 since kp >= 8... TB <= 256)
  const int col = tid / P, sub = tid % P;
  double acc = 0.0;
  __syncthreads();
  for (int64_t t0 = (int64_t)lb * TB; t0 < n; t0 += (int64_t)S.gps * TB) {
    const int64_t e = t0 + tid;
    const bool in = e < n;
    if (in) {
      const double* p = V + o0 + e;
      for (int i = 0; i < k; ++i) cpa8(sv + (size_t)i * SV + tid, p + (size_t)i * ldv);
    }
    cp_commit_v();
    double wv = in ? w[o0 + e] : 0.0;
    cp_wait_all_v();
    if (MODE != 0) {
      double s0 = 0.0, s1 = 0.0;
      if (in) {
        int i = 0;
        for (; i + 1 < k; i += 2) {
          s0 += cf[i] * sv[(size_t)i * SV + tid];
          s1 += cf[i + 1] * sv[(size_t)(i + 1) * SV + tid];
        }
        if (i < k) s0 += cf[i] * sv[(size_t)i * SV + tid];
        wv -= s0 + s1;
        if (MODE == 1) w[o0 + e] = wv;
        else vout[o0 + e] = wv;
      }
      if (MODE == 2) acc += wv * wv;
    }
    if (MODE != 2) {
      if (!in)
        for (int i = 0; i < k; ++i) sv[(size_t)i * SV + tid] = 0.0;
      sw[tid] = wv;
      __syncthreads();
      if (col < k) {
        const double* c = sv + (size_t)col * SV;
        for (int q = sub; q < TB; q += P) acc += c[q] * sw[q];
      }
      __syncthreads();
    }
  }
  // block reduction -> partial[blockIdx.x * pld + i]
  if (MODE == 2) {
    double v = warp_sum(acc);
    if (lane == 0) cs[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < TB / 32; ++q) t += cs[q];
      partial[(size_t)blockIdx.x * pld] = t;
    }
  } else {
    for (int o = P >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (sub == 0 && col < k) partial[(size_t)blockIdx.x * pld + col] = acc;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(counters + s, 1u) == (unsigned)S.gps - 1u);
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int kout = MODE == 2 ? 1 : k;
  for (int i = warp; i < kout; i += TB / 32) {
    const double a = partial_sum(partial, (size_t)s * S.gps, pld, S.gps, i, lane);
    if (lane == 0) out[(size_t)s * ldo + i] = (MODE != 2 && sc) ? a * sc[(size_t)s * lds + i] : a;
  }
  if (tid == 0) counters[s] = 0u;
}

// ---------------------------------------------------------------- DCGS2 passes
// Delayed CGS2 (krylov.cu): per Arnoldi step one reduction pass and one update
// pass over the basis.  Columns staged per tile: Q_0 .. Q_{j-1} and the lagged
// vector u_j = V_j (k = j + 1 columns); z = A u_j streamed alongside.
//   k_dcgs_dots:   out[i] = <col_i, u_j>,  out[k + i] = <col_i, z>   (i < k)
//   k_dcgs_update: V_j <- (u_j - sum_i b_i Q_i) / rho
//                  V_{j+1} <- (z - mu u_j - sum_i e_i Q_i) / rho
//   (b = coef[0..j), e = coef[ldc .. ldc + j), rho = coef[2 ldc], mu = coef[2 ldc + 1];
//   segment s reads coef + s * cstride)
// L2 prefetch of the 16-byte granules inside [p, p + n) doubles (bulk; rounded
// inward at the end, the start rounds down by < 16 bytes into the same vector).
__device__ __forceinline__ void prefetch_l2(const double* p, int64_t n) {
  const uintptr_t a0 = (uintptr_t)p & ~(uintptr_t)15;
  const uintptr_t a1 = (uintptr_t)(p + n) & ~(uintptr_t)15;
  if (n <= 0 || a1 <= a0) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a0), "r"((unsigned)(a1 - a0))
               : "memory");
}

__device__ __forceinline__ void cp_wait_pending(int n) {  // all but the newest n groups
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
  }
}

// Threads per column P and the stage layout of k_dcgs_dots: element e of a tile
// column sits at (e % P) * R + e / P, R = TB / P + 2, so the elements one thread
// sums (e = sub, sub + P, ...) are adjacent (16-byte loads) and the cp.async
// writes of a warp spread over the banks; a column takes P * R = TB + 2P doubles.
__host__ __device__ inline int dots_threads_per_col(int TB, int k) {
  int kp = 8;
  while (kp < k) kp <<= 1;
  return kp >= TB ? 1 : TB / kp;
}

// Tiles are staged through a ring of ns stages (ns = 1..4, chosen by the launcher
// from k): the copies of the next ns - 1 tiles are in flight while a tile's
// column dots run.  Per thread the tiles and elements are summed in the same
// order for every ns and layout.
struct NoEpi {
  __device__ void operator()(int) const {}
};
// Epi: run by every thread of the block that finishes the reduction of segment s,
// after out[s * ldo + 0 .. 2k) is written (e.g. the GMRES step that consumes it).
template <int TB, class Epi = NoEpi>
static __global__ void __launch_bounds__(TB) k_dcgs_dots(Seg S, int k, const double* __restrict__ V,
                                                         int64_t ldv, const double* __restrict__ z,
                                                         double* partial, int pld, double* out,
                                                         int ldo, unsigned* counters,
                                                         const int* __restrict__ skip, int ns,
                                                         Epi epi = Epi()) {
  pdl_wait();
  pdl_trigger();
  if (skip && *skip) return;
  extern __shared__ double smp[];  // ns stages of k + 1 columns (Q_0 .. Q_{j-1}, u_j, z)
  __shared__ bool last;
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = dots_threads_per_col(TB, k);
  const int M = TB / P, R = M + 2, SV = TB + 2 * P;
  const int col = tid / P, sub = tid % P;
  const int pos = (tid % P) * R + tid / P;  // where this thread's element is staged
  const size_t stage = (size_t)(k + 1) * SV;
  const int64_t stride = (int64_t)S.gps * TB;
  auto issue = [&](int64_t t0, double* buf) {
    const int64_t e = t0 + tid;
    if (e < n) {
      const double* p = V + o0 + e;
      for (int i = 0; i < k; ++i) cpa8(buf + (size_t)i * SV + pos, p + (size_t)i * ldv);
      cpa8(buf + (size_t)k * SV + pos, z + o0 + e);
    } else if (t0 < n) {
      for (int i = 0; i <= k; ++i) buf[(size_t)i * SV + pos] = 0.0;
    }
    cp_commit_v();  // one group per tile, possibly empty
  };
  const int64_t tfirst = (int64_t)lb * TB;
  for (int q = 0; q < ns - 1; ++q) issue(tfirst + q * stride, smp + (size_t)q * stage);
  double a1 = 0.0, a2 = 0.0;
  // k > TB (only TB = 128 with GMRES(128): k = 129 at the cycle's last step): P = 1 and
  // thread tid also owns column col2 = tid + TB (same element order as every column)
  const int col2 = col + TB;
  double b1 = 0.0, b2 = 0.0;
  int it = 0;
  for (int64_t t0 = tfirst; t0 < n; t0 += stride, ++it) {
    issue(t0 + (int64_t)(ns - 1) * stride, smp + (size_t)((it + ns - 1) % ns) * stage);
    {  // the tile after the ring window: into L2 while this one is reduced
      const int64_t tp = t0 + (int64_t)ns * stride;  // (1 or 2 tiles further: slower)
      if (tid <= k && tp < n) prefetch_l2((tid < k ? V + (size_t)tid * ldv : z) + o0 + tp, min((int64_t)TB, n - tp));
    }
    cp_wait_pending(ns - 1);
    __syncthreads();
    const double* sv = smp + (size_t)(it % ns) * stage;
    if (col < k) {
      const double2* c = (const double2*)(sv + (size_t)col * SV + sub * R);
      const double2* su = (const double2*)(sv + (size_t)(k - 1) * SV + sub * R);  // lagged u_j
      const double2* sz = (const double2*)(sv + (size_t)k * SV + sub * R);
      for (int m = 0; m < M / 2; ++m) {  // elements sub + P (2m), sub + P (2m + 1)
        const double2 cv = c[m], uv = su[m], zv = sz[m];
        a1 += cv.x * uv.x;
        a2 += cv.x * zv.x;
        a1 += cv.y * uv.y;
        a2 += cv.y * zv.y;
      }
    }
    if (col2 < k) {  // P == 1 here
      const double2* c = (const double2*)(sv + (size_t)col2 * SV + sub * R);
      const double2* su = (const double2*)(sv + (size_t)(k - 1) * SV + sub * R);
      const double2* sz = (const double2*)(sv + (size_t)k * SV + sub * R);
      for (int m = 0; m < M / 2; ++m) {
        const double2 cv = c[m], uv = su[m], zv = sz[m];
        b1 += cv.x * uv.x;
        b2 += cv.x * zv.x;
        b1 += cv.y * uv.y;
        b2 += cv.y * zv.y;
      }
    }
    __syncthreads();
  }
  cp_wait_all_v();
  for (int o = P >> 1; o > 0; o >>= 1) {
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (sub == 0 && col < k) {
    partial[(size_t)blockIdx.x * pld + col] = a1;
    partial[(size_t)blockIdx.x * pld + k + col] = a2;
  }
  if (col2 < k) {
    partial[(size_t)blockIdx.x * pld + col2] = b1;
    partial[(size_t)blockIdx.x * pld + k + col2] = b2;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(counters + s, 1u) == (unsigned)S.gps - 1u);
  __syncthreads();
  if (!last) return;
  __threadfence();
  constexpr int NW = TB / 32;
  for (int i = warp; i < 2 * k; i += 2 * NW) {  // two columns per warp at a time
    const int i2 = i + NW;
    if (i2 < 2 * k) {
      double a, a2;
      partial_sum2(partial, (size_t)s * S.gps, pld, S.gps, i, i2, lane, a, a2);
      if (lane == 0) {
        out[(size_t)s * ldo + i] = a;
        out[(size_t)s * ldo + i2] = a2;
      }
    } else {
      const double a = partial_sum(partial, (size_t)s * S.gps, pld, S.gps, i, lane);
      if (lane == 0) out[(size_t)s * ldo + i] = a;
    }
  }
  if (tid == 0) counters[s] = 0u;
  __syncthreads();  // out[] written by this block is visible to all its threads
  epi(s);
}

// ---- bulk-copy (TMA engine) variant of the reduction pass:
// one thread arms an mbarrier with the tile's byte count and issues one
// cp.async.bulk per column (2 KB) instead of one 8-byte cp.async per element;
// the others wait on the mbarrier.  Column i of a stage at i * (TB + 4); every
// thread sums the same elements in the same order as k_dcgs_dots's original
// layout (bit-identical results).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <class Epi = NoEpi>
static __global__ void __launch_bounds__(256) k_dcgs_dots_bulk(Seg S, int k, const double* __restrict__ V,
                                                               int64_t ldv, const double* __restrict__ z,
                                                               double* partial, int pld, double* out,
                                                               int ldo, unsigned* counters,
                                                               const int* __restrict__ skip, int ns,
                                                               Epi epi = Epi()) {
  constexpr int TB = 256, SVB = TB + 4;
  pdl_wait();
  pdl_trigger();
  if (skip && *skip) return;
  extern __shared__ __align__(16) double smp[];
  __shared__ __align__(8) uint64_t full[4];
  __shared__ bool last;
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = dots_threads_per_col(TB, k);
  const int col = tid / P, sub = tid % P;
  const size_t stage = (size_t)(k + 1) * SVB;
  const int64_t stride = (int64_t)S.gps * TB;
  if (tid == 0) {
    for (int q = 0; q < ns; ++q) mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // A segment starting at an odd element is copied from one element earlier
  // (16-byte aligned source) and read at offset sh = 1 in the stage.
  const int sh = (int)(o0 & 1);
  auto issue = [&](int64_t t0, int q) {  // thread 0
    if (t0 >= n) return;
    const int cnt = (int)min((int64_t)TB, n - t0) + sh;
    const unsigned bytes = (unsigned)((cnt + 1) & ~1) * 8u;  // 16-byte granules (padded vectors)
    double* dst = smp + (size_t)q * stage;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(&full[q], bytes * (unsigned)(k + 1));
    for (int i = 0; i < k; ++i)
      bulk_g2s(dst + (size_t)i * SVB, V + (size_t)i * ldv + o0 - sh + t0, bytes, &full[q]);
    bulk_g2s(dst + (size_t)k * SVB, z + o0 - sh + t0, bytes, &full[q]);
  };
  const int64_t tfirst = (int64_t)lb * TB;
  if (tid == 0)
    for (int q = 0; q < ns - 1; ++q) issue(tfirst + q * stride, q);
  double a1 = 0.0, a2 = 0.0;
  unsigned ph = 0;
  int it = 0;
  for (int64_t t0 = tfirst; t0 < n; t0 += stride, ++it) {
    const int q = it % ns;
    if (tid == 0) issue(t0 + (int64_t)(ns - 1) * stride, (it + ns - 1) % ns);
    {  // the tile after the ring window: into L2 while this one is reduced
      const int64_t tp = t0 + (int64_t)ns * stride;
      if (tid <= k && tp < n) prefetch_l2((tid < k ? V + (size_t)tid * ldv : z) + o0 + tp, min((int64_t)TB, n - tp));
    }
    mbar_wait(&full[q], (ph >> q) & 1u);
    ph ^= 1u << q;
    double* sv = smp + (size_t)q * stage + sh;
    if (t0 + TB > n) {  // the last tile: elements past n read as 0 (as the staged zeros of k_dcgs_dots)
      if (t0 + tid >= n)
        for (int i = 0; i <= k; ++i) sv[(size_t)i * SVB + tid] = 0.0;
      __syncthreads();
    }
    if (col < k) {
      const double* c = sv + (size_t)col * SVB;
      const double* su = sv + (size_t)(k - 1) * SVB;  // the lagged vector is the last column
      const double* sz = sv + (size_t)k * SVB;
      for (int e = sub; e < TB; e += P) {
        const double cv = c[e];
        a1 += cv * su[e];
        a2 += cv * sz[e];
      }
    }
    __syncthreads();  // the stage is refilled by the next issue
  }
  for (int o = P >> 1; o > 0; o >>= 1) {
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (sub == 0 && col < k) {
    partial[(size_t)blockIdx.x * pld + col] = a1;
    partial[(size_t)blockIdx.x * pld + k + col] = a2;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(counters + s, 1u) == (unsigned)S.gps - 1u);
  __syncthreads();
  if (!last) return;
  __threadfence();
  constexpr int NW = TB / 32;
  for (int i = warp; i < 2 * k; i += 2 * NW) {
    const int i2 = i + NW;
    if (i2 < 2 * k) {
      double a, a2v;
      partial_sum2(partial, (size_t)s * S.gps, pld, S.gps, i, i2, lane, a, a2v);
      if (lane == 0) {
        out[(size_t)s * ldo + i] = a;
        out[(size_t)s * ldo + i2] = a2v;
      }
    } else {
      const double a = partial_sum(partial, (size_t)s * S.gps, pld, S.gps, i, lane);
      if (lane == 0) out[(size_t)s * ldo + i] = a;
    }
  }
  if (tid == 0) counters[s] = 0u;
  __syncthreads();
  epi(s);
}

// ---- register-direct variant of the reduction pass: every basis column is read
// ONCE from HBM straight into registers (coalesced 16-byte loads, no shared-memory
// staging).  Warp w of the block owns the columns i = w, w + 8, ... (< k) and keeps
// their two partial dots <Q_i, u_j>, <Q_i, z> per lane; a tile is 128 consecutive
// elements, lane l taking elements 2l, 2l+1, 64+2l, 65+2l; every warp also reads the
// tile's u_j and z (L1 hits after the first warp).  Fixed association order: per
// lane the tiles in order, then the warp shuffle tree, then the blocks in index
// order (the last block of the segment, as k_dcgs_dots).  KW = max columns per warp.
// ---- TMA-staged variant with warp-owned columns (single 16-byte aligned segment):
// tiles of 128 elements; one thread arms an mbarrier and issues one cp.async.bulk
// per column (Q_0 .. Q_{k-1} (the last is u_j), z) into a ring of ns stages, so up
// to ns tiles' columns are in flight without occupying registers; warp w reduces
// its columns w, w+8, ... of a staged tile with 16-byte shared loads (lane l:
// elements 2l, 2l+1, 64+2l, 65+2l), u_j and z of the tile held in registers.
// Same per-lane element order and epilogue as k_dcgs_dots_direct.
template <int KW, class Epi = NoEpi>
static __global__ void __launch_bounds__(256, 2) k_dcgs_dots_tma(Seg S, int k, const double* __restrict__ V,
                                                                  int64_t ldv, const double* __restrict__ z,
                                                                  double* partial, int pld, double* out, int ldo,
                                                                  unsigned* counters, const int* __restrict__ skip,
                                                                  int ns, Epi epi = Epi()) {
  constexpr int TB = 256, NW = TB / 32, TE = 128;
  pdl_wait();
  pdl_trigger();
  if (skip && *skip) return;
  extern __shared__ __align__(16) double smt[];
  __shared__ __align__(8) uint64_t full[8];
  __shared__ bool last;
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t stage = (size_t)(k + 1) * TE;
  const int64_t stride = (int64_t)S.gps * TE;
  if (tid == 0) {
    for (int q = 0; q < ns; ++q) mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t t0, int q) {  // thread 0
    if (t0 >= n) return;
    const unsigned bytes = (unsigned)((min((int64_t)TE, n - t0) + 1) & ~1) * 8u;  // 16-byte granules
    double* dst = smt + (size_t)q * stage;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(&full[q], bytes * (unsigned)(k + 1));
    for (int i = 0; i < k; ++i) bulk_g2s(dst + (size_t)i * TE, V + (size_t)i * ldv + o0 + t0, bytes, &full[q]);
    bulk_g2s(dst + (size_t)k * TE, z + o0 + t0, bytes, &full[q]);
  };
  const int64_t tfirst = (int64_t)lb * TE;
  if (tid == 0)
    for (int q = 0; q < ns - 1; ++q) issue(tfirst + q * stride, q);
  double a1[KW], a2[KW];
#pragma unroll
  for (int c = 0; c < KW; ++c) a1[c] = a2[c] = 0.0;
  unsigned ph = 0;
  int it = 0;
  for (int64_t t0 = tfirst; t0 < n; t0 += stride, ++it) {
    const int q = it % ns;
    if (tid == 0) issue(t0 + (int64_t)(ns - 1) * stride, (it + ns - 1) % ns);
    mbar_wait(&full[q], (ph >> q) & 1u);
    ph ^= 1u << q;
    const double* sv = smt + (size_t)q * stage;
    const int e0 = 2 * lane, e1 = 64 + 2 * lane;
    const bool ok0 = t0 + e0 < n, ok1 = t0 + e0 + 1 < n, ok2 = t0 + e1 < n, ok3 = t0 + e1 + 1 < n;
    const double2 ua = *(const double2*)(sv + (size_t)(k - 1) * TE + e0), ub = *(const double2*)(sv + (size_t)(k - 1) * TE + e1);
    const double2 za = *(const double2*)(sv + (size_t)k * TE + e0), zb = *(const double2*)(sv + (size_t)k * TE + e1);
    const double u0 = ok0 ? ua.x : 0.0, u1 = ok1 ? ua.y : 0.0, u2 = ok2 ? ub.x : 0.0, u3 = ok3 ? ub.y : 0.0;
    const double z0 = ok0 ? za.x : 0.0, z1 = ok1 ? za.y : 0.0, z2 = ok2 ? zb.x : 0.0, z3 = ok3 ? zb.y : 0.0;
#pragma unroll
    for (int c = 0; c < KW; ++c) {
      const int i = warp + c * NW;
      if (i < k) {
        const double2 va = *(const double2*)(sv + (size_t)i * TE + e0), vb = *(const double2*)(sv + (size_t)i * TE + e1);
        const double v0 = ok0 ? va.x : 0.0, v1 = ok1 ? va.y : 0.0, v2 = ok2 ? vb.x : 0.0, v3 = ok3 ? vb.y : 0.0;
        a1[c] = fma(v0, u0, a1[c]); a2[c] = fma(v0, z0, a2[c]);
        a1[c] = fma(v1, u1, a1[c]); a2[c] = fma(v1, z1, a2[c]);
        a1[c] = fma(v2, u2, a1[c]); a2[c] = fma(v2, z2, a2[c]);
        a1[c] = fma(v3, u3, a1[c]); a2[c] = fma(v3, z3, a2[c]);
      }
    }
    __syncthreads();  // the stage is refilled by the next issue
  }
#pragma unroll
  for (int c = 0; c < KW; ++c) {
    const int i = warp + c * NW;
    if (i < k) {
      const double r1 = warp_sum(a1[c]), r2 = warp_sum(a2[c]);
      if (lane == 0) {
        partial[(size_t)blockIdx.x * pld + i] = r1;
        partial[(size_t)blockIdx.x * pld + k + i] = r2;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(counters + s, 1u) == (unsigned)S.gps - 1u);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = warp; i < 2 * k; i += 2 * NW) {
    const int i2 = i + NW;
    if (i2 < 2 * k) {
      double a, a2v;
      partial_sum2(partial, (size_t)s * S.gps, pld, S.gps, i, i2, lane, a, a2v);
      if (lane == 0) {
        out[(size_t)s * ldo + i] = a;
        out[(size_t)s * ldo + i2] = a2v;
      }
    } else {
      const double a = partial_sum(partial, (size_t)s * S.gps, pld, S.gps, i, lane);
      if (lane == 0) out[(size_t)s * ldo + i] = a;
    }
  }
  if (tid == 0) counters[s] = 0u;
  __syncthreads();
  epi(s);
}

template <int KW, int MINB, int UN, class Epi = NoEpi>
static __global__ void __launch_bounds__(256, MINB) k_dcgs_dots_direct(
    Seg S, int k, const double* __restrict__ V, int64_t ldv, const double* __restrict__ z, double* partial,
    int pld, double* out, int ldo, unsigned* counters, const int* __restrict__ skip, Epi epi = Epi()) {
  constexpr int TB = 256, NW = TB / 32, TE = 128;
  pdl_wait();
  pdl_trigger();
  if (skip && *skip) return;
  __shared__ bool last;
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* uj = V + (size_t)(k - 1) * ldv + o0;  // the lagged vector is the last column
  const double* zz = z + o0;
  double a1[KW], a2[KW];
#pragma unroll
  for (int c = 0; c < KW; ++c) a1[c] = a2[c] = 0.0;
  const bool vec2 = ((o0 | ldv) & 1) == 0;  // 16-byte aligned columns
  const int64_t stride = (int64_t)S.gps * TE;
  // UN tiles per iteration (all their loads issued before the FMAs); per lane the
  // tiles are still summed in increasing order
  // UN > 0: UN tiles per iteration, one column's loads at a time; UN <= 0: max(1, -UN)
  // tiles per iteration with every owned column's loads issued before the FMAs
  constexpr int UQ = UN > 0 ? UN : (UN == 0 ? 1 : -UN);
  for (int64_t tb = (int64_t)lb * TE; tb < n; tb += UQ * stride) {
    double u[UQ][4], zv[UQ][4];
#pragma unroll
    for (int q = 0; q < UQ; ++q) {
      const int64_t t0 = tb + q * stride;
      const int64_t e0 = t0 + 2 * lane, e1 = t0 + 64 + 2 * lane;
      if (t0 + TE <= n && vec2) {
        const double2 ua = __ldg((const double2*)(uj + e0)), ub = __ldg((const double2*)(uj + e1));
        const double2 za = __ldg((const double2*)(zz + e0)), zb = __ldg((const double2*)(zz + e1));
        u[q][0] = ua.x; u[q][1] = ua.y; u[q][2] = ub.x; u[q][3] = ub.y;
        zv[q][0] = za.x; zv[q][1] = za.y; zv[q][2] = zb.x; zv[q][3] = zb.y;
      } else {
        u[q][0] = e0 < n ? __ldg(uj + e0) : 0.0; u[q][1] = e0 + 1 < n ? __ldg(uj + e0 + 1) : 0.0;
        u[q][2] = e1 < n ? __ldg(uj + e1) : 0.0; u[q][3] = e1 + 1 < n ? __ldg(uj + e1 + 1) : 0.0;
        zv[q][0] = e0 < n ? __ldg(zz + e0) : 0.0; zv[q][1] = e0 + 1 < n ? __ldg(zz + e0 + 1) : 0.0;
        zv[q][2] = e1 < n ? __ldg(zz + e1) : 0.0; zv[q][3] = e1 + 1 < n ? __ldg(zz + e1 + 1) : 0.0;
      }
    }
    if (UN <= 0) {  // every owned column's loads of the UQ tiles issued before the FMAs
      double v[UQ][KW][4];
#pragma unroll
      for (int q = 0; q < UQ; ++q) {
        const int64_t t0 = tb + q * stride;
        const int64_t e0 = t0 + 2 * lane, e1 = t0 + 64 + 2 * lane;
        const bool fv = t0 + TE <= n && vec2;
#pragma unroll
        for (int c = 0; c < KW; ++c) {
          const int i = warp + c * NW;
          const double* col = V + (size_t)min(i, k - 1) * ldv + o0;
          if (fv) {
            const double2 va = __ldcs((const double2*)(col + e0)), vb = __ldcs((const double2*)(col + e1));
            v[q][c][0] = va.x; v[q][c][1] = va.y; v[q][c][2] = vb.x; v[q][c][3] = vb.y;
          } else {
            v[q][c][0] = e0 < n ? __ldcs(col + e0) : 0.0; v[q][c][1] = e0 + 1 < n ? __ldcs(col + e0 + 1) : 0.0;
            v[q][c][2] = e1 < n ? __ldcs(col + e1) : 0.0; v[q][c][3] = e1 + 1 < n ? __ldcs(col + e1 + 1) : 0.0;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < UQ; ++q)
#pragma unroll
        for (int c = 0; c < KW; ++c)
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            a1[c] = fma(v[q][c][x], u[q][x], a1[c]);
            a2[c] = fma(v[q][c][x], zv[q][x], a2[c]);
          }
      continue;
    }
#pragma unroll
    for (int c = 0; c < KW; ++c) {
      const int i = warp + c * NW;
      if (i < k) {
        const double* col = V + (size_t)i * ldv + o0;
        double v[UQ][4];
#pragma unroll
        for (int q = 0; q < UQ; ++q) {
          const int64_t t0 = tb + q * stride;
          const int64_t e0 = t0 + 2 * lane, e1 = t0 + 64 + 2 * lane;
          if (t0 + TE <= n && vec2) {
            const double2 va = __ldcs((const double2*)(col + e0)), vb = __ldcs((const double2*)(col + e1));
            v[q][0] = va.x; v[q][1] = va.y; v[q][2] = vb.x; v[q][3] = vb.y;
          } else {
            v[q][0] = e0 < n ? __ldcs(col + e0) : 0.0; v[q][1] = e0 + 1 < n ? __ldcs(col + e0 + 1) : 0.0;
            v[q][2] = e1 < n ? __ldcs(col + e1) : 0.0; v[q][3] = e1 + 1 < n ? __ldcs(col + e1 + 1) : 0.0;
          }
        }
#pragma unroll
        for (int q = 0; q < UQ; ++q)
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            a1[c] = fma(v[q][x], u[q][x], a1[c]);
            a2[c] = fma(v[q][x], zv[q][x], a2[c]);
          }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < KW; ++c) {
    const int i = warp + c * NW;
    if (i < k) {
      const double r1 = warp_sum(a1[c]), r2 = warp_sum(a2[c]);
      if (lane == 0) {
        partial[(size_t)blockIdx.x * pld + i] = r1;
        partial[(size_t)blockIdx.x * pld + k + i] = r2;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(counters + s, 1u) == (unsigned)S.gps - 1u);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = warp; i < 2 * k; i += 2 * NW) {
    const int i2 = i + NW;
    if (i2 < 2 * k) {
      double a, a2v;
      partial_sum2(partial, (size_t)s * S.gps, pld, S.gps, i, i2, lane, a, a2v);
      if (lane == 0) {
        out[(size_t)s * ldo + i] = a;
        out[(size_t)s * ldo + i2] = a2v;
      }
    } else {
      const double a = partial_sum(partial, (size_t)s * S.gps, pld, S.gps, i, lane);
      if (lane == 0) out[(size_t)s * ldo + i] = a;
    }
  }
  if (tid == 0) counters[s] = 0u;
  __syncthreads();
  epi(s);
}

template <int TB>
static __global__ void __launch_bounds__(TB) k_dcgs_update(Seg S, int k, double* V, int64_t ldv,
                                                           const double* __restrict__ z,
                                                           const double* __restrict__ coef0, int ldc,
                                                           int64_t cstride, const int* __restrict__ skip) {
  pdl_wait();
  if (skip && *skip) return;
  constexpr int SV = TB + 4;
  extern __shared__ double smp[];
  double* sv = smp;             // k columns of SV
  double* cb = sv + (size_t)k * SV;
  double* ce = cb + k;
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  const double* coef = coef0 + (size_t)s * cstride;  // this segment's coefficients
  const int tid = threadIdx.x;
  const int j = k - 1;
  for (int i = tid; i < j; i += TB) {
    cb[i] = coef[i];
    ce[i] = coef[ldc + i];
  }
  const double rinv = 1.0 / coef[2 * ldc], mu = coef[2 * ldc + 1];
  __syncthreads();
  // tiles from the block's last to its first: the reduction pass before this one
  // ended on the high tiles, which are still in L2 (each element is independent)
  const int64_t stride = (int64_t)S.gps * TB, tf = (int64_t)lb * TB;
  const int64_t tl = tf < n ? tf + (n - 1 - tf) / stride * stride : tf - stride;
  for (int64_t t0 = tl; t0 >= tf; t0 -= stride) {
    const int64_t e = t0 + tid;
    if (e >= n) continue;
    const double* p = V + o0 + e;
    for (int i = 0; i < k; ++i) cpa8(sv + (size_t)i * SV + tid, p + (size_t)i * ldv);
    cp_commit_v();
    const double zv = z[o0 + e];
    cp_wait_all_v();
    double sb0 = 0.0, sb1 = 0.0, se0 = 0.0, se1 = 0.0;
    int i = 0;
    for (; i + 1 < j; i += 2) {
      const double q0 = sv[(size_t)i * SV + tid], q1 = sv[(size_t)(i + 1) * SV + tid];
      sb0 += cb[i] * q0;
      sb1 += cb[i + 1] * q1;
      se0 += ce[i] * q0;
      se1 += ce[i + 1] * q1;
    }
    if (i < j) {
      const double q0 = sv[(size_t)i * SV + tid];
      sb0 += cb[i] * q0;
      se0 += ce[i] * q0;
    }
    const double uv = sv[(size_t)j * SV + tid];
    V[(size_t)j * ldv + o0 + e] = (uv - (sb0 + sb1)) * rinv;
    V[(size_t)(j + 1) * ldv + o0 + e] = (zv - mu * uv - (se0 + se1)) * rinv;
  }
}

// The same update with the basis elements loaded straight into registers (a
// thread only ever uses its own element of each column): k - 1 <= KMAX, no
// shared-memory staging; identical arithmetic order.
template <int TB, int KMAX, int MINB = 2>
static __global__ void __launch_bounds__(TB, MINB) k_dcgs_update_reg(Seg S, int k, double* V, int64_t ldv,
                                                                  const double* __restrict__ z,
                                                                  const double* __restrict__ coef0,
                                                                  int ldc, int64_t cstride,
                                                                  const int* __restrict__ skip) {
  __shared__ double cb[KMAX], ce[KMAX];
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  const int tid = threadIdx.x;
  const int j = k - 1;
  // tiles from the block's last to its first: the reduction pass before this one
  // ended on the high tiles, which are still in L2 (each element is independent)
  const int64_t stride = (int64_t)S.gps * TB, tf = (int64_t)lb * TB;
  const int64_t tl = tf < n ? tf + (n - 1 - tf) / stride * stride : tf - stride;
  // the first tile's Q columns, u_j and z are loaded before pdl_wait(): they were
  // written two or more kernels back (the apply before the reduction pass this
  // kernel follows, the update passes before it), so only the coefficients wait
  double q[KMAX], uv = 0.0, zv = 0.0;
  {
    const int64_t e = tl + tid;
    if (tl >= tf && e < n) {
      const double* p = V + o0 + e;
#pragma unroll
      for (int i = 0; i < KMAX; ++i)
        if (i < j) q[i] = __ldcg(p + (size_t)i * ldv);
      uv = __ldcg(p + (size_t)j * ldv);
      zv = __ldcg(z + o0 + e);
    }
  }
  pdl_wait();
  if (skip && *skip) return;
  const double* coef = coef0 + (size_t)s * cstride;  // this segment's coefficients
  for (int i = tid; i < j; i += TB) {
    cb[i] = coef[i];
    ce[i] = coef[ldc + i];
  }
  const double rinv = 1.0 / coef[2 * ldc], mu = coef[2 * ldc + 1];
  __syncthreads();
  for (int64_t t0 = tl; t0 >= tf; t0 -= stride) {
    const int64_t e = t0 + tid;
    if (e >= n) continue;
    if (t0 != tl) {
      const double* p = V + o0 + e;
#pragma unroll
      for (int i = 0; i < KMAX; ++i)
        if (i < j) q[i] = __ldcg(p + (size_t)i * ldv);
      uv = __ldcg(p + (size_t)j * ldv);
      zv = __ldcg(z + o0 + e);
    }
    double sb0 = 0.0, sb1 = 0.0, se0 = 0.0, se1 = 0.0;
#pragma unroll
    for (int i = 0; i + 1 < KMAX; i += 2) {
      if (i + 1 < j) {
        sb0 += cb[i] * q[i];
        sb1 += cb[i + 1] * q[i + 1];
        se0 += ce[i] * q[i];
        se1 += ce[i + 1] * q[i + 1];
      } else if (i < j) {  // odd j: the last column
        sb0 += cb[i] * q[i];
        se0 += ce[i] * q[i];
      }
    }
    if ((KMAX & 1) && KMAX - 1 < j) {  // unreachable for the even KMAX used
      sb0 += cb[KMAX - 1] * q[KMAX - 1];
      se0 += ce[KMAX - 1] * q[KMAX - 1];
    }
    V[(size_t)j * ldv + o0 + e] = (uv - (sb0 + sb1)) * rinv;
    V[(size_t)(j + 1) * ldv + o0 + e] = (zv - mu * uv - (se0 + se1)) * rinv;
  }
}

template <int TB>
inline size_t proj_smem(int k) {
  return ((size_t)k * (TB + 4) + TB + (size_t)k + TB / 32) * sizeof(double);
}

// w <- w - sum_i coef_i sc_i V_i ;  out_i = sc_i <V_i, w_new>   (per segment)
template <int KMAX>
static __global__ void __launch_bounds__(VB) k_cgs_update(Seg S, int k, const double* __restrict__ V,
                                                   int64_t ldv, double* __restrict__ w,
                                                   const double* __restrict__ sc, int lds,
                                                   const double* __restrict__ coef, double* partial,
                                                   double* out, int ldo, unsigned* counters) {
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  __shared__ double cf[KMAX];
  for (int i = threadIdx.x; i < k; i += VB) cf[i] = coef[(size_t)s * ldo + i] * sc[(size_t)s * lds + i];
  __syncthreads();
  double acc[KMAX];
#pragma unroll
  for (int i = 0; i < KMAX; ++i) acc[i] = 0.0;
  for (int64_t e = (int64_t)lb * VB + threadIdx.x; e < n; e += (int64_t)S.gps * VB) {
    const double* p = V + o0 + e;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int i = 0; i < KMAX; i += 4) {
      if (i < k) s0 += cf[i] * __ldg(p + (size_t)i * ldv);
      if (i + 1 < k) s1 += cf[i + 1] * __ldg(p + (size_t)(i + 1) * ldv);
      if (i + 2 < k) s2 += cf[i + 2] * __ldg(p + (size_t)(i + 2) * ldv);
      if (i + 3 < k) s3 += cf[i + 3] * __ldg(p + (size_t)(i + 3) * ldv);
    }
    const double wv = w[o0 + e] - ((s0 + s1) + (s2 + s3));
    w[o0 + e] = wv;
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < k) acc[i] += __ldg(p + (size_t)i * ldv) * wv;   // L1/L2 re-read
  }
  block_then_segment_reduce<KMAX>(acc, k, partial, KMAX, s, S.gps, sc, lds, out, ldo, counters);
}

// vout <- w - sum_i coef_i sc_i V_i ; out = ||vout||^2 (per segment). vout may alias w.
static __global__ void __launch_bounds__(VB) k_cgs_final(Seg S, int k, const double* __restrict__ V,
                                                  int64_t ldv, const double* w,
                                                  const double* __restrict__ sc, int lds,
                                                  const double* __restrict__ coef, int ldo,
                                                  double* vout, double* partial, double* out,
                                                  int ldn, unsigned* counters) {
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  __shared__ double cf[132];
  for (int i = threadIdx.x; i < k; i += VB) cf[i] = coef[(size_t)s * ldo + i] * sc[(size_t)s * lds + i];
  __syncthreads();
  double acc[1] = {0.0};
  for (int64_t e = (int64_t)lb * VB + threadIdx.x; e < n; e += (int64_t)S.gps * VB) {
    const double* p = V + o0 + e;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int i = 0;
    for (; i + 3 < k; i += 4) {
      s0 += cf[i] * __ldcs(p + (size_t)i * ldv);
      s1 += cf[i + 1] * __ldcs(p + (size_t)(i + 1) * ldv);
      s2 += cf[i + 2] * __ldcs(p + (size_t)(i + 2) * ldv);
      s3 += cf[i + 3] * __ldcs(p + (size_t)(i + 3) * ldv);
    }
    for (; i < k; ++i) s0 += cf[i] * __ldcs(p + (size_t)i * ldv);
    const double v = w[o0 + e] - ((s0 + s1) + (s2 + s3));
    vout[o0 + e] = v;
    acc[0] += v * v;
  }
  block_then_segment_reduce<1>(acc, 1, partial, 1, s, S.gps, nullptr, 0, out, ldn, counters);
}

// out = b - t (t may be null), ||out||^2 per segment into res[s*ldr]. out may be null.
static __global__ void __launch_bounds__(VB) k_sub_nrm2(Seg S, const double* __restrict__ b,
                                                 const double* __restrict__ t, double* out,
                                                 double* partial, double* res, int ldr,
                                                 unsigned* counters) {
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  double acc[1] = {0.0};
  for (int64_t e = (int64_t)lb * VB + threadIdx.x; e < n; e += (int64_t)S.gps * VB) {
    const double v = b[o0 + e] - (t ? t[o0 + e] : 0.0);
    if (out) out[o0 + e] = v;
    acc[0] += v * v;
  }
  block_then_segment_reduce<1>(acc, 1, partial, 1, s, S.gps, nullptr, 0, res, ldr, counters);
}

// x[dst] += sum_{i<k_s} y_si * sc_si * V_i[src]  over a per-segment element range
// [lo_s, hi_s) of V (src = o0 + lo + q) written to xo[xoff_s + q].
// coefs: y at ys[s*ldy + i], sc at sc[s*lds + i] (sc may be null), k_s at ks[s] or k.
static __global__ void __launch_bounds__(VB) k_combine(Seg S, const double* __restrict__ V, int64_t ldv,
                                                const double* __restrict__ ys, int ldy,
                                                const double* __restrict__ sc, int lds,
                                                const int* ks, int ks_ld, int kfix,
                                                const int64_t* lo, const int64_t* hi,
                                                const int64_t* xoff, double* __restrict__ x,
                                                int accumulate) {
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s];
  const int64_t a = lo ? lo[s] : 0, bnd = hi ? hi[s] : (S.off[s + 1] - o0);
  const int64_t xo = xoff ? xoff[s] : o0;
  const int k = ks ? ks[(size_t)s * ks_ld] : kfix;
  __shared__ double cf[130];
  for (int i = threadIdx.x; i < k; i += VB)
    cf[i] = ys[(size_t)s * ldy + i] * (sc ? sc[(size_t)s * lds + i] : 1.0);
  __syncthreads();
  for (int64_t q = a + (int64_t)lb * VB + threadIdx.x; q < bnd; q += (int64_t)S.gps * VB) {
    const double* p = V + o0 + q;
    double s0 = 0.0, s1 = 0.0;
    int i = 0;
    for (; i + 1 < k; i += 2) {
      s0 += cf[i] * __ldg(p + (size_t)i * ldv);
      s1 += cf[i + 1] * __ldg(p + (size_t)(i + 1) * ldv);
    }
    if (i < k) s0 += cf[i] * __ldg(p + (size_t)i * ldv);
    const int64_t d = xo + (q - a);
    x[d] = (accumulate ? x[d] : 0.0) + (s0 + s1);
  }
}

// y = sc_s[idx] * x per segment (scale pointer per segment: sc[s*lds + idx])
static __global__ void __launch_bounds__(VB) k_scale(Seg S, const double* __restrict__ x,
                                              const double* __restrict__ sc, int lds, int idx,
                                              double* __restrict__ y) {
  const int s = blockIdx.x / S.gps, lb = blockIdx.x % S.gps;
  const int64_t o0 = S.off[s], n = S.off[s + 1] - o0;
  const double f = sc[(size_t)s * lds + idx];
  for (int64_t e = (int64_t)lb * VB + threadIdx.x; e < n; e += (int64_t)S.gps * VB)
    y[o0 + e] = f * x[o0 + e];
}

}  // namespace vec

// Launch helpers choosing the register-array width from k.
int launch_mdot(const vec::Seg& S, int k, const double* V, int64_t ldv, const double* w,
                const double* sc, int lds, double* partial, double* out, int ldo,
                unsigned* counters, cudaStream_t st);  // k <= kMaxRestart + 2
int launch_cgs_update(const vec::Seg& S, int k, const double* V, int64_t ldv, double* w,
                      const double* sc, int lds, const double* coef, double* partial, double* out,
                      int ldo, unsigned* counters, cudaStream_t st);
int launch_cgs_final(const vec::Seg& S, int k, const double* V, int64_t ldv, const double* w,
                     const double* sc, int lds, const double* coef, int ldo, double* vout,
                     double* partial, double* out, int ldn, unsigned* counters, cudaStream_t st);
// delayed CGS2 passes (k = j + 1 columns: Q_0..Q_{j-1} and the lagged u_j)
int launch_dcgs_dots(const vec::Seg& S, int k, const double* V, int64_t ldv, const double* z,
                     double* partial, int pld, double* out, int ldo, unsigned* counters,
                     cudaStream_t st, const int* skip = nullptr);
int launch_dcgs_update(const vec::Seg& S, int k, double* V, int64_t ldv, const double* z,
                       const double* coef, int ldc, int64_t cstride, cudaStream_t st,
                       const int* skip = nullptr);

// The reduction pass with an epilogue run by the block that completes each
// segment's reduction (vec::k_dcgs_dots).
template <class Epi>
inline int launch_dcgs_dots_epi(const vec::Seg& S, int k, const double* V, int64_t ldv, const double* z,
                                double* partial, int pld, double* out, int ldo, unsigned* counters,
                                cudaStream_t st, const int* skip, Epi epi) {
  const int grid = S.nseg * S.gps;
  // ring depth: up to 4 stages within ~110 KB (2 blocks per SM)
  auto depth = [](size_t stage) { return (int)std::max<size_t>(1, std::min<size_t>(4, (110 * 1024) / stage)); };
  static const bool bulk = [] {  // CPM_DOTS_BULK=0: the per-element cp.async kernel (A/B)
    const char* v = getenv("CPM_DOTS_BULK");
    return !v || *v != '0';
  }();
  static const bool direct_env = [] {  // CPM_DOTS_DIRECT=0: the staged kernels (A/B)
    const char* v = getenv("CPM_DOTS_DIRECT");
    return !v || *v != '0';
  }();
  // the register-direct kernel for the single-segment (global) GMRES and for aligned
  // segments (the RAS inner solves pad each segment to 32 elements); unaligned
  // segments: the bulk-staged kernel
  const bool direct = direct_env && (S.nseg == 1 || S.aligned);
  // register-direct reduction pass: every owned column's loads of a tile issued
  // before its FMAs (UN = 0), columns per warp KW by k (fewer registers for small k)
  // CPM_DOTS_TMA=1: the TMA-staged variant (measured slower: 42.3 against 33.1 ms per
  // 204 passes of a config-1 solve; the per-tile block barrier of the ring) — A/B only
  static const bool tma = [] {
    const char* v = getenv("CPM_DOTS_TMA");
    return v && *v == '1';
  }();
  if (direct && tma && k <= 8 * 17) {
    // ring depth: up to 8 stages within ~100 KB (two blocks per SM); one stage (no
    // overlap inside the block) when a stage alone exceeds that (k > 96)
    const size_t stage = (size_t)(k + 1) * 128 * sizeof(double);
    const int ns = (int)std::max<size_t>(1, std::min<size_t>(8, (100 * 1024) / stage));
    static bool attr[4] = {false, false, false, false};  // per kernel variant
    auto run = [&](auto kern, int v) -> int {
      if (!attr[v]) {
        CPM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr[v] = true;
      }
      CPM_CUDA(launch_pdl(kern, dim3(grid), dim3(256), ns * stage, st, S, k, V, ldv, z, partial, pld, out, ldo,
                          counters, skip, ns, epi));
      return CPM_OK;
    };
    if (k <= 8 * 2) CPM_TRY(run(vec::k_dcgs_dots_tma<2, Epi>, 0));
    else if (k <= 8 * 4) CPM_TRY(run(vec::k_dcgs_dots_tma<4, Epi>, 1));
    else if (k <= 8 * 8) CPM_TRY(run(vec::k_dcgs_dots_tma<8, Epi>, 2));
    else CPM_TRY(run(vec::k_dcgs_dots_tma<17, Epi>, 3));
    count_launch();
    CPM_CUDA(cudaGetLastError());
    return CPM_OK;
  }
  static const int tt = [] {  // CPM_DOTS_TT=1: one tile per iteration also for k <= 32 (A/B)
    const char* v = getenv("CPM_DOTS_TT");
    return v ? atoi(v) : 2;
  }();
  if (direct && k <= 8 * 2 && tt == 2) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_dots_direct<2, 2, -3, Epi>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z,
                        partial, pld, out, ldo, counters, skip, epi));
  } else if (direct && k <= 8 * 4 && tt == 2) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_dots_direct<4, 2, -2, Epi>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z,
                        partial, pld, out, ldo, counters, skip, epi));
  } else if (direct && k <= 8 * 2) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_dots_direct<2, 2, 0, Epi>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z,
                        partial, pld, out, ldo, counters, skip, epi));
  } else if (direct && k <= 8 * 4) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_dots_direct<4, 2, 0, Epi>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z,
                        partial, pld, out, ldo, counters, skip, epi));
  } else if (direct && k <= 8 * 6) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_dots_direct<6, 2, 0, Epi>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z,
                        partial, pld, out, ldo, counters, skip, epi));
  } else if (direct && k <= 8 * 8) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_dots_direct<8, 2, 0, Epi>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z,
                        partial, pld, out, ldo, counters, skip, epi));
  } else if (direct && k <= 8 * 17) {
    CPM_CUDA(launch_pdl(vec::k_dcgs_dots_direct<17, 2, 1, Epi>, dim3(grid), dim3(256), 0, st, S, k, V, ldv, z,
                        partial, pld, out, ldo, counters, skip, epi));
  } else if (bulk && k <= 52) {  // a stage of (k+1) 2 KB columns: two blocks per SM
    const size_t stage = (size_t)(k + 1) * (256 + 4) * sizeof(double);
    const int ns = depth(stage);
    static bool attrb = false;
    if (!attrb) {
      CPM_CUDA(cudaFuncSetAttribute(vec::k_dcgs_dots_bulk<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    200 * 1024));
      attrb = true;
    }
    CPM_CUDA(launch_pdl(vec::k_dcgs_dots_bulk<Epi>, dim3(grid), dim3(256), ns * stage, st, S, k, V, ldv,
                        z, partial, pld, out, ldo, counters, skip, ns, epi));
  } else if (k <= 51) {  // CPM_DOTS_BULK=0 (A/B)
    const size_t stage = (size_t)(k + 1) * (256 + 2 * vec::dots_threads_per_col(256, k)) * sizeof(double);
    const int ns = depth(stage);
    static bool attr = false;
    if (!attr) {
      CPM_CUDA(cudaFuncSetAttribute(vec::k_dcgs_dots<256, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    200 * 1024));
      attr = true;
    }
    CPM_CUDA(launch_pdl(vec::k_dcgs_dots<256, Epi>, dim3(grid), dim3(256), ns * stage, st, S, k, V, ldv,
                        z, partial, pld, out, ldo, counters, skip, ns, epi));
  } else {
    const size_t stage = (size_t)(k + 1) * (128 + 2 * vec::dots_threads_per_col(128, k)) * sizeof(double);
    const int ns = depth(stage);
    static bool attr = false;
    if (!attr) {
      CPM_CUDA(cudaFuncSetAttribute(vec::k_dcgs_dots<128, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    200 * 1024));
      attr = true;
    }
    vec::k_dcgs_dots<128, Epi><<<grid, 128, ns * stage, st>>>(S, k, V, ldv, z, partial, pld, out, ldo,
                                                              counters, skip, ns, epi);
  }
  count_launch();
  CPM_CUDA(cudaGetLastError());
  return CPM_OK;
}

}  // namespace cpm
