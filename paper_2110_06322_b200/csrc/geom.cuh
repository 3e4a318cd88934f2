// geom.cuh — closest point functions and lattice/Morton helpers (device + host).
//
// The band membership test (dist <= lambda) and the stencil base floor(cp/h)
// are integer decisions taken from floating point; reading R3 of DESIGN.md fixes
// the operation order so that they are reproducible: every product, quotient,
// sum and square root below is an explicitly round-to-nearest IEEE binary64
// operation (no contraction into FMA), sums are evaluated left to right.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.cuh"

namespace cpm {

#ifdef __CUDA_ARCH__
#define RN_ADD(a, b) __dadd_rn((a), (b))
#define RN_SUB(a, b) __dsub_rn((a), (b))
#define RN_MUL(a, b) __dmul_rn((a), (b))
#define RN_DIV(a, b) __ddiv_rn((a), (b))
#define RN_SQRT(a) __dsqrt_rn((a))
#else
#define RN_ADD(a, b) ((a) + (b))
#define RN_SUB(a, b) ((a) - (b))
#define RN_MUL(a, b) ((a) * (b))
#define RN_DIV(a, b) ((a) / (b))
#define RN_SQRT(a) sqrt((a))
#endif

// cp_S(x) and |x - cp_S(x)| (Eq. 3).  Returns false where cp is
// undefined (sphere centre, torus axis / core circle); dist is then +inf.
__host__ __device__ inline bool closest_point(const Surface& s, double x, double y, double z,
                                              double* cx, double* cy, double* cz, double* dist) {
  if (s.kind == CPM_SURF_SPHERE) {
    const double R = s.p[0];
    double r = RN_SQRT(RN_ADD(RN_ADD(RN_MUL(x, x), RN_MUL(y, y)), RN_MUL(z, z)));
    if (r == 0.0) {
      *dist = INFINITY;
      return false;
    }
    *cx = RN_DIV(RN_MUL(R, x), r);
    *cy = RN_DIV(RN_MUL(R, y), r);
    *cz = RN_DIV(RN_MUL(R, z), r);
    *dist = fabs(RN_SUB(r, R));
    return true;
  } else {  // torus about z
    const double R = s.p[0], rr = s.p[1];
    double rho = RN_SQRT(RN_ADD(RN_MUL(x, x), RN_MUL(y, y)));
    if (rho == 0.0) {
      *dist = INFINITY;
      return false;
    }
    double qx = RN_DIV(RN_MUL(R, x), rho);
    double qy = RN_DIV(RN_MUL(R, y), rho);
    double dx = RN_SUB(x, qx), dy = RN_SUB(y, qy), dz = z;
    double dn = RN_SQRT(RN_ADD(RN_ADD(RN_MUL(dx, dx), RN_MUL(dy, dy)), RN_MUL(dz, dz)));
    if (dn == 0.0) {
      *dist = INFINITY;
      return false;
    }
    *cx = RN_ADD(qx, RN_DIV(RN_MUL(rr, dx), dn));
    *cy = RN_ADD(qy, RN_DIV(RN_MUL(rr, dy), dn));
    *cz = RN_DIV(RN_MUL(rr, dz), dn);
    *dist = fabs(RN_SUB(dn, rr));
    return true;
  }
}

__host__ __device__ inline double surface_dist(const Surface& s, double x, double y, double z) {
  double a, b, c, d;
  closest_point(s, x, y, z, &a, &b, &c, &d);
  return d;
}

// Lattice point x = i * h (one rounded product, reading R3).
__host__ __device__ inline double lat(int i, double h) { return RN_MUL((double)i, h); }

// floor(i / 8) and i mod 8 for signed lattice indices.
__host__ __device__ inline int brick_of(int i) { return ((i + (kMortonBias << 3)) >> 3) - kMortonBias; }
__host__ __device__ inline int local_of(int i) { return i - (brick_of(i) << 3); }

__host__ __device__ inline uint64_t part1by2(uint64_t x) {
  x &= 0x1fffffull;
  x = (x | (x << 32)) & 0x1f00000000ffffull;
  x = (x | (x << 16)) & 0x1f0000ff0000ffull;
  x = (x | (x << 8)) & 0x100f00f00f00f00full;
  x = (x | (x << 4)) & 0x10c30c30c30c30c3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}
__host__ __device__ inline uint64_t compact1by2(uint64_t x) {
  x &= 0x1249249249249249ull;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ull;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00full;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffull;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffull;
  x = (x ^ (x >> 32)) & 0x1fffffull;
  return x;
}
// Morton code of a brick (reading R8): bit b of x -> 3b, y -> 3b+1, z -> 3b+2.
__host__ __device__ inline uint64_t brick_morton(int bx, int by, int bz) {
  return part1by2((uint64_t)(bx + kMortonBias)) | (part1by2((uint64_t)(by + kMortonBias)) << 1) |
         (part1by2((uint64_t)(bz + kMortonBias)) << 2);
}
__host__ __device__ inline void morton_brick(uint64_t m, int* bx, int* by, int* bz) {
  *bx = (int)compact1by2(m) - kMortonBias;
  *by = (int)compact1by2(m >> 1) - kMortonBias;
  *bz = (int)compact1by2(m >> 2) - kMortonBias;
}

}  // namespace cpm
