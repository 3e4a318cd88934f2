// apply.cu — matrix-free stabilised CPM operator (north_star item 2).
//
//   y = c u - [Delta_h E u - (6/h^2)(u - E u)]          (Eq. 4, d = 3)
//     = (c + 6/h^2) u - (1/h^2) sum_{6 nbrs j} (E u)_j    (the centre (E u)_i terms cancel)
//
// Two kernels per apply, one CTA per tile (= occupied 8^3 brick):
//   extend  : stage the tile's 4x4x4-stencil box of u in shared memory (fill
//             runs of consecutive band-order sources), then for every eval node
//             (Sigma_A u Sigma_G in the brick) recompute the tricubic Lagrange
//             weights from its fractional offsets and contract
//             x, then y, then z.  E u is written to a dense per-brick scratch vb.
//   laplace : for every output node, 6 neighbour reads of vb (same brick or a
//             face-neighbour brick) and the diagonal term.
// HBM-bound by design (no tensor cores: this is a gather, not a dense
// contraction).  Bytes per apply: DESIGN.md §"Roofline".
#include "internal.cuh"

namespace cpm {
namespace {

// Degree-3 Lagrange weights on nodes (-1, 0, 1, 2) at t (product form).
__device__ __forceinline__ void lagrange4(double t, double w[4]) {
  const double a = t + 1.0, c = t - 1.0, d = t - 2.0;
  const double cd = c * d, at = a * t;
  w[0] = -(t * cd) * (1.0 / 6.0);
  w[1] = (a * cd) * 0.5;
  w[2] = -(at * d) * 0.5;
  w[3] = (at * c) * (1.0 / 6.0);
}

template <bool ZERO>
__global__ void __launch_bounds__(256) k_extend(const TileHdr* __restrict__ tiles,
                                                const uint64_t* __restrict__ runs,
                                                const double* __restrict__ u,
                                                const double* __restrict__ tx,
                                                const double* __restrict__ ty,
                                                const double* __restrict__ tz,
                                                const uint32_t* __restrict__ eoff,
                                                double* __restrict__ vb) {
  extern __shared__ double box[];
  const int t = blockIdx.x;
  const TileHdr* T = tiles + t;
  const int e0 = T->e0, e1 = T->e1, r0 = T->r0, r1 = T->r1;
  const int sx = T->sx, sxy = T->sx * T->sy;
  if (ZERO) {
    const int nbox = sxy * T->sz;
    for (int c = threadIdx.x; c < nbox; c += blockDim.x) box[c] = 0.0;
    __syncthreads();
  }
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const uint64_t run = __ldg(runs + r);
    const uint32_t src = (uint32_t)run, dst = (uint32_t)(run >> 32) & 0xffffu,
                   len = (uint32_t)(run >> 48) & 0xffu;
    for (uint32_t q = 0; q < len; ++q) box[dst + q] = __ldg(u + src + q);
  }
  __syncthreads();
  double* out = vb + (size_t)t * kBrickCells;
  for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    double wx[4], wy[4], wz[4];
    lagrange4(__ldg(tx + e), wx);
    lagrange4(__ldg(ty + e), wy);
    lagrange4(__ldg(tz + e), wz);
    const uint32_t eo = __ldg(eoff + e);
    const double* p = box + (eo & 0xffffu);
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double accy = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double* row = p + b * sx + c * sxy;
        const double rx = wx[0] * row[0] + wx[1] * row[1] + wx[2] * row[2] + wx[3] * row[3];
        accy += wy[b] * rx;
      }
      acc += wz[c] * accy;
    }
    out[eo >> 16] = acc;
  }
}

__global__ void __launch_bounds__(256) k_laplace(const TileHdr* __restrict__ tiles,
                                                 const double* __restrict__ u,
                                                 const uint16_t* __restrict__ acell,
                                                 const double* __restrict__ vb,
                                                 double* __restrict__ y, double diag, double ih2,
                                                 const double* __restrict__ scale) {
  const int t = blockIdx.x;
  const TileHdr* T = tiles + t;
  const int a0 = T->a0, a1 = T->a1;
  if (a0 == a1) return;
  const int n0 = T->nbr[0], n1 = T->nbr[1], n2 = T->nbr[2], n3 = T->nbr[3], n4 = T->nbr[4],
            n5 = T->nbr[5];
  const double* vt = vb + (size_t)t * kBrickCells;
  const double s = scale ? __ldg(scale) : 1.0;
  for (int a = a0 + threadIdx.x; a < a1; a += blockDim.x) {
    const int c = __ldg(acell + a);
    const int lx = c & 7, ly = (c >> 3) & 7, lz = c >> 6;
    double sum;
    sum = (lx < 7) ? vt[c + 1] : vb[(size_t)n0 * kBrickCells + c - 7];
    sum += (lx > 0) ? vt[c - 1] : vb[(size_t)n1 * kBrickCells + c + 7];
    sum += (ly < 7) ? vt[c + 8] : vb[(size_t)n2 * kBrickCells + c - 56];
    sum += (ly > 0) ? vt[c - 8] : vb[(size_t)n3 * kBrickCells + c + 56];
    sum += (lz < 7) ? vt[c + 64] : vb[(size_t)n4 * kBrickCells + c - 448];
    sum += (lz > 0) ? vt[c - 64] : vb[(size_t)n5 * kBrickCells + c + 448];
    y[a] = s * (diag * __ldg(u + a) - ih2 * sum);
  }
}

bool g_attr_set = false;

}  // namespace

int apply_device(const cpm_band* b, double c, const double* u, double* y, const double* scale,
                 cudaStream_t s) {
  if (!g_attr_set) {
    CPM_CUDA(cudaFuncSetAttribute(k_extend<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kMaxBoxCells * (int)sizeof(double)));
    CPM_CUDA(cudaFuncSetAttribute(k_extend<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kMaxBoxCells * (int)sizeof(double)));
    g_attr_set = true;
  }
  const size_t smem = (size_t)b->maxBox * sizeof(double);
  const double ih2 = 1.0 / (b->h * b->h);
  const double diag = c + 6.0 * ih2;
  {
    ProfScope ps(K_EXTEND, s);
    if (b->zeroFill)
      k_extend<true><<<b->nT, 256, smem, s>>>(b->tiles, b->runs, u, b->tx, b->ty, b->tz, b->eoff,
                                              b->vb);
    else
      k_extend<false><<<b->nT, 256, smem, s>>>(b->tiles, b->runs, u, b->tx, b->ty, b->tz, b->eoff,
                                               b->vb);
    count_launch();
  }
  {
    ProfScope ps(K_LAPLACE, s);
    k_laplace<<<b->nT, 256, 0, s>>>(b->tiles, u, b->acell, b->vb, y, diag, ih2, scale);
    count_launch();
  }
  CPM_CUDA(cudaGetLastError());
  return CPM_OK;
}

}  // namespace cpm
