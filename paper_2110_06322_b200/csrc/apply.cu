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
#include <algorithm>

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

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int kExtThreads = 256;
constexpr int kExtMinBlocks = 4;   // CTAs per SM the register budget is sized for
constexpr int kNodesPerThread = 2; // eval nodes per tile <= 512 = 2 * kExtThreads

// Issue the asynchronous copies of tile t's stencil box (fill runs, 8 lanes per
// run; cp.async = LDGSTS).  ZERO: clear the box first.
template <bool ZERO>
__device__ __forceinline__ void stage_box(const TileHdr* __restrict__ tiles,
                                          const uint64_t* __restrict__ runs,
                                          const double* __restrict__ u,
                                          const double* __restrict__ uh, uint32_t split, int t,
                                          double* box) {
  const TileHdr* T = tiles + t;
  const int r0 = T->r0, r1 = T->r1;
  if (ZERO) {
    const int nbox = T->pad[1] * T->sz;
    for (int c = threadIdx.x; c < nbox; c += kExtThreads) box[c] = 0.0;
    __syncthreads();
  }
  // Thread-per-run: all run descriptors of the tile are loaded up front (4 per
  // thread in flight), then each thread issues the LDGSTS copies of its runs.
  // (A dependent descriptor->copy chain per loop trip was the kernel's main stall.)
  const int nr = r1 - r0;
  for (int base = 0; base < nr; base += 4 * kExtThreads) {
    uint64_t d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = base + threadIdx.x + k * kExtThreads;
      d[k] = r < nr ? __ldg(runs + r0 + r) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t src = (uint32_t)d[k], dst = (uint32_t)(d[k] >> 32) & 0xffffu,
                     len = (uint32_t)(d[k] >> 48) & 0xffu;
      const double* gsrc = src >= split ? uh + (src - split) : u + src;  // runs never straddle split
      for (uint32_t q = 0; q < len; ++q) cp_async8(box + dst + q, gsrc + q);
    }
  }
}

struct NodeRegs {
  double t[kNodesPerThread][3];
  uint32_t eo[kNodesPerThread];
  int n;
};

__device__ __forceinline__ void load_nodes(const TileHdr* __restrict__ tiles,
                                           const double* __restrict__ tx,
                                           const double* __restrict__ ty,
                                           const double* __restrict__ tz,
                                           const uint32_t* __restrict__ eoff, int t, NodeRegs& R) {
  const int e0 = tiles[t].e0, ne = tiles[t].e1 - e0;
  R.n = ne;
#pragma unroll
  for (int k = 0; k < kNodesPerThread; ++k) {
    const int i = threadIdx.x + k * kExtThreads;
    if (i < ne) {
      R.t[k][0] = __ldg(tx + e0 + i);
      R.t[k][1] = __ldg(ty + e0 + i);
      R.t[k][2] = __ldg(tz + e0 + i);
      R.eo[k] = __ldg(eoff + e0 + i);
    }
  }
}

// Persistent extend: CTA b handles tiles b, b + G, b + 2G, ...  While tile t is
// contracted, tile t + G's stencil box streams into the other shared-memory
// buffer (cp.async) and its node offsets into registers, so the global-memory
// latency of one tile overlaps the FP64 / shared-memory work of the previous.
template <bool ZERO>
__global__ void __launch_bounds__(kExtThreads, kExtMinBlocks)
    k_extend(const TileHdr* __restrict__ tiles, int nT, int boxCells,
             const uint64_t* __restrict__ runs, const double* __restrict__ u,
             const double* __restrict__ uh, uint32_t split,
             const double* __restrict__ tx, const double* __restrict__ ty,
             const double* __restrict__ tz, const uint32_t* __restrict__ eoff,
             double* __restrict__ vb) {
  extern __shared__ double smem[];
  int t = blockIdx.x;
  if (t >= nT) return;
  NodeRegs cur, nxt;
  stage_box<ZERO>(tiles, runs, u, uh, split, t, smem);
  cp_commit();
  load_nodes(tiles, tx, ty, tz, eoff, t, cur);
  int b = 0;
  for (; t < nT; t += gridDim.x) {
    const int tn = t + gridDim.x;
    if (tn < nT) {
      stage_box<ZERO>(tiles, runs, u, uh, split, tn, smem + (size_t)(b ^ 1) * boxCells);
      load_nodes(tiles, tx, ty, tz, eoff, tn, nxt);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const double* box = smem + (size_t)b * boxCells;
    const TileHdr* T = tiles + t;
    const int sx = T->pad[0], sxy = T->pad[1];
    double* out = vb + (size_t)t * kBrickCells;
#pragma unroll
    for (int k = 0; k < kNodesPerThread; ++k) {
      if (threadIdx.x + k * kExtThreads < cur.n) {
        double wx[4], wy[4], wz[4];
        lagrange4(cur.t[k][0], wx);
        lagrange4(cur.t[k][1], wy);
        lagrange4(cur.t[k][2], wz);
        const uint32_t eo = cur.eo[k];
        const double* p = box + (eo & 0xffffu);
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double accy = 0.0;
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) {
            const double* row = p + bb * sx + c * sxy;
            const double rx = wx[0] * row[0] + wx[1] * row[1] + wx[2] * row[2] + wx[3] * row[3];
            accy += wy[bb] * rx;
          }
          acc += wz[c] * accy;
        }
        out[eo >> 16] = acc;
      }
    }
    __syncthreads();  // buffer b is refilled by the next iteration's prefetch
    cur = nxt;
    b ^= 1;
  }
  cp_wait<0>();
}

__global__ void __launch_bounds__(256) k_laplace(const TileHdr* __restrict__ tiles,
                                                 const double* __restrict__ u,
                                                 const uint16_t* __restrict__ acell,
                                                 const double* __restrict__ vb,
                                                 double* __restrict__ y, double diag, double ih2,
                                                 const double* __restrict__ scale, int lds) {
  const int t = blockIdx.x;
  const TileHdr* T = tiles + t;
  const int a0 = T->a0, a1 = T->a1;
  if (a0 == a1) return;
  const int n0 = T->nbr[0], n1 = T->nbr[1], n2 = T->nbr[2], n3 = T->nbr[3], n4 = T->nbr[4],
            n5 = T->nbr[5];
  const double* vt = vb + (size_t)t * kBrickCells;
  const double s = scale ? __ldg(scale + (size_t)T->pad[2] * lds) : 1.0;
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
int g_sms = 0;

}  // namespace

int apply_device(const cpm_band* b, double c, const double* u, double* y, const double* scale,
                 int lds, cudaStream_t s) {
  return apply_device_split(b, c, u, u, y, scale, lds, s);
}

int apply_device_split(const cpm_band* b, double c, const double* u, const double* uh, double* y,
                       const double* scale, int lds, cudaStream_t s) {
  const size_t smemMax = 2 * (size_t)kMaxBoxCells * sizeof(double);
  if (!g_attr_set) {
    CPM_CUDA(cudaFuncSetAttribute(k_extend<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smemMax));
    CPM_CUDA(cudaFuncSetAttribute(k_extend<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smemMax));
    int dev = 0;
    CPM_CUDA(cudaGetDevice(&dev));
    CPM_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    g_attr_set = true;
  }
  const size_t smem = 2 * (size_t)b->maxBox * sizeof(double);
  // CTAs per SM limited by shared memory (227 KB usable) and the launch bound
  const int per_sm = std::max(1, std::min<int>(kExtMinBlocks, (int)((227 * 1024) / (smem + 1024))));
  const int grid = std::max(1, std::min(b->nT, g_sms * per_sm));
  const double ih2 = 1.0 / (b->h * b->h);
  const double diag = c + 6.0 * ih2;
  {
    ProfScope ps(K_EXTEND, s);
    if (b->zeroFill)
      k_extend<true><<<grid, kExtThreads, smem, s>>>(b->tiles, b->nT, b->maxBox, b->runs, u, uh,
                                                     b->srcSplit, b->tx, b->ty, b->tz, b->eoff, b->vb);
    else
      k_extend<false><<<grid, kExtThreads, smem, s>>>(b->tiles, b->nT, b->maxBox, b->runs, u, uh,
                                                      b->srcSplit, b->tx, b->ty, b->tz, b->eoff, b->vb);
    count_launch();
  }
  {
    ProfScope ps(K_LAPLACE, s);
    k_laplace<<<b->nT, 256, 0, s>>>(b->tiles, u, b->acell, b->vb, y, diag, ih2, scale, lds);
    count_launch();
  }
  CPM_CUDA(cudaGetLastError());
  return CPM_OK;
}

}  // namespace cpm
