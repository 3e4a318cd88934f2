// ras.cu — one-level restricted additive Schwarz with batched inexact local GMRES
// (north_star item 4, Dirichlet transmission PAPER.md:105,252).
//
//   z = M r = sum_j R~_j^T  GMRES_k(A_j, R_j r),   A_j = R_j A R_j^T
//
// Setup (all on the GPU):
//   * active 6-neighbour table from the tiles' occupancy masks;
//   * subdomain membership as one bit per subdomain per node: slab bits
//     (reading R8), then `overlap` growth sweeps over the neighbour table (R7);
//   * one "multi-band": the concatenation over subdomains of sub-tiles (every
//     global tile holding a member node or face-adjacent to one), with output
//     ranges in the concatenated local numbering, per-tile segment id, and
//     stencil-box fill runs restricted to members (cells outside S_j read 0);
//     the eval-node geometry (offsets, box offsets) is shared with the band.
// Apply (no host synchronisation): gather R_j r for all j at once, k steps of
// CGS2 Arnoldi on all segments in lockstep (segmented kernels of vecops.cuh and
// the same extend/laplace kernels as the global operator), per-segment Givens
// least squares, and a combine that writes only the disjoint part of each
// subdomain (restricted prolongation) straight into z.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "geom.cuh"
#include "krylov.cuh"
#include "part.cuh"
#include "ras.cuh"
#include "vecops.cuh"

namespace cpm {
namespace {

constexpr int VB = vec::VB;

__device__ inline bool mhas(const uint32_t* m16, int cell) { return (m16[cell >> 5] >> (cell & 31)) & 1u; }
__device__ inline int mrank(const uint32_t* m16, int cell) {
  int w = cell >> 5, r = 0;
  for (int q = 0; q < w; ++q) r += __popc(m16[q]);
  return r + __popc(m16[w] & ((1u << (cell & 31)) - 1u));
}

// active node index of (tile, cell) or -1
__device__ inline int active_at(const TileHdr* tiles, const uint32_t* amask, int tile, int cell) {
  if (tile < 0) return -1;
  const uint32_t* m = amask + (size_t)tile * 16;
  if (!mhas(m, cell)) return -1;
  return tiles[tile].a0 + mrank(m, cell);
}

__global__ void k_nbr_active(const TileHdr* tiles, const uint32_t* amask, const uint16_t* acell,
                             int* nbr) {
  const int t = blockIdx.x;
  const TileHdr T = tiles[t];
  for (int a = T.a0 + threadIdx.x; a < T.a1; a += blockDim.x) {
    const int c = acell[a];
    const int lx = c & 7, ly = (c >> 3) & 7, lz = c >> 6;
    int* o = nbr + 6 * (size_t)a;
    o[0] = lx < 7 ? active_at(tiles, amask, t, c + 1) : active_at(tiles, amask, T.nbr[0], c - 7);
    o[1] = lx > 0 ? active_at(tiles, amask, t, c - 1) : active_at(tiles, amask, T.nbr[1], c + 7);
    o[2] = ly < 7 ? active_at(tiles, amask, t, c + 8) : active_at(tiles, amask, T.nbr[2], c - 56);
    o[3] = ly > 0 ? active_at(tiles, amask, t, c - 8) : active_at(tiles, amask, T.nbr[3], c + 56);
    o[4] = lz < 7 ? active_at(tiles, amask, t, c + 64) : active_at(tiles, amask, T.nbr[4], c - 448);
    o[5] = lz > 0 ? active_at(tiles, amask, t, c - 64) : active_at(tiles, amask, T.nbr[5], c + 448);
  }
}

__host__ __device__ inline int64_t slab_lo(int s, int64_t n, int S) { return ((int64_t)s * n) / S; }

__global__ void k_member_init(int64_t n, int S, uint64_t* bits) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n;
       a += (int64_t)gridDim.x * blockDim.x) {
    int s = (int)((a * S) / n);
    while (s + 1 < S && slab_lo(s + 1, n, S) <= a) ++s;
    while (s > 0 && slab_lo(s, n, S) > a) --s;
    bits[a] = 1ull << s;
  }
}

__global__ void k_member_grow(int64_t n, const int* nbr, const uint64_t* in, uint64_t* out) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n;
       a += (int64_t)gridDim.x * blockDim.x) {
    uint64_t b = in[a];
    for (int d = 0; d < 6; ++d) {
      const int q = nbr[6 * a + d];
      if (q >= 0) b |= in[q];
    }
    out[a] = b;
  }
}

__global__ void k_flag_bit(int64_t n, const uint64_t* bits, int s, int* flag) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a <= n;
       a += (int64_t)gridDim.x * blockDim.x)
    flag[a] = (a < n) ? (int)((bits[a] >> s) & 1ull) : 0;
}

__global__ void k_tile_has(const TileHdr* tiles, const uint64_t* bits, int s, int* has) {
  const int t = blockIdx.x;
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  const TileHdr T = tiles[t];
  for (int a = T.a0 + threadIdx.x; a < T.a1; a += blockDim.x)
    if ((bits[a] >> s) & 1ull) any = 1;
  __syncthreads();
  if (threadIdx.x == 0) has[t] = any;
}

__global__ void k_tile_include(int nT, const TileHdr* tiles, const int* has, int* inc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > nT) return;
  if (t == nT) {
    inc[t] = 0;
    return;
  }
  int v = has[t];
  for (int d = 0; d < 6 && !v; ++d) {
    const int q = tiles[t].nbr[d];
    if (q >= 0 && has[q]) v = 1;
  }
  inc[t] = v;
}

__global__ void k_subtiles(int nT, const TileHdr* tiles, const int* inc, const int* incpos,
                           const int* pos, int64_t loff, int toff, int s, TileHdr* sub,
                           int* tmap) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nT) return;
  if (!inc[t]) {
    tmap[t] = -1;
    return;
  }
  const int q = incpos[t];
  tmap[t] = toff + q;
  TileHdr T = tiles[t];
  T.a0 = (int32_t)(loff + pos[tiles[t].a0]);
  T.a1 = (int32_t)(loff + pos[tiles[t].a1]);
  T.pad[2] = s;
  sub[toff + q] = T;
}

__global__ void k_subtile_nbrs(int n, TileHdr* sub, const int* tmap) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  for (int d = 0; d < 6; ++d) {
    const int g = sub[q].nbr[d];
    sub[q].nbr[d] = g >= 0 ? tmap[g] : -1;
  }
}

__global__ void k_local_index(int64_t n, const int* flag, const int* pos, int64_t loff,
                              const uint16_t* acell, int64_t* gidx, uint16_t* acl) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n;
       a += (int64_t)gridDim.x * blockDim.x)
    if (flag[a]) {
      gidx[loff + pos[a]] = a;
      acl[loff + pos[a]] = acell[a];
    }
}

__device__ inline int bmap_at(const int* bmap, const int* blo, const int* bdim, int bx, int by,
                              int bz) {
  const int x = bx - blo[0], y = by - blo[1], z = bz - blo[2];
  if (x < 0 || y < 0 || z < 0 || x >= bdim[0] || y >= bdim[1] || z >= bdim[2]) return -1;
  return bmap[((size_t)z * bdim[1] + y) * bdim[0] + x];
}

__global__ void k_rows(int n, const TileHdr* sub, int64_t* nrows) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) nrows[q] = (int64_t)sub[q].sy * sub[q].sz;
  if (q == 0) nrows[n] = 0;
}

// Fill runs of the sub-tiles of one subdomain: thread per (sub-tile, box row);
// maximal segments of consecutive member cells inside one brick row.
template <bool WRITE>
__global__ void k_sub_runs(const TileHdr* sub, const TileHdr* tiles, const uint32_t* amask,
                           const int* bmap, const int* blo, const int* bdim, const uint64_t* bits,
                           int s, const int* pos, int64_t loff, const int64_t* rowbase,
                           int64_t* rowcnt, const int64_t* runstart, uint64_t* runs, int64_t zsrc) {
  const int q = blockIdx.x;
  const TileHdr T = sub[q];
  const int nrows = T.sy * T.sz;
  for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
    const int y = T.oy + r % T.sy, z = T.oz + r / T.sy;
    const int by = brick_of(y), bz = brick_of(z), ly = local_of(y), lz = local_of(z);
    const int64_t gi = rowbase[q] + r;
    const int64_t out = WRITE ? runstart[gi] : 0;
    int64_t n = 0;
    int x = T.ox;
    const int xe = T.ox + T.sx;
    while (x < xe) {
      const int bx = brick_of(x);
      const int xend = min(xe, bx * 8 + 8);
      const int g = bmap_at(bmap, blo, bdim, bx, by, bz);
      if (g >= 0) {
        const uint32_t* m = amask + (size_t)g * 16;
        int lq = local_of(x);
        const int lxe = xend - bx * 8;
        while (lq < lxe) {
          const int cell = lq + 8 * ly + 64 * lz;
          const int a = mhas(m, cell) ? tiles[g].a0 + mrank(m, cell) : -1;
          if (a < 0) {  // not in Sigma_A: no stencil reads it
            ++lq;
            continue;
          }
          if (!((bits[a] >> s) & 1ull)) {
            // Sigma_A cells outside the subdomain: a run from the zero source (src =
            // zsrc reads the apply's zero buffer; with zsrc < 0 the box is cleared)
            const int q0 = lq;
            ++lq;
            while (lq < lxe && mhas(m, lq + 8 * ly + 64 * lz) && !((bits[a + (lq - q0)] >> s) & 1ull)) ++lq;
            if (zsrc >= 0) {
              if (WRITE) {
                const uint32_t dst =
                    (uint32_t)((bx * 8 + q0 - T.ox) + T.pad[0] * (y - T.oy) + T.pad[1] * (z - T.oz));
                runs[out + n] = pack_run((uint32_t)zsrc, dst, (uint32_t)(lq - q0));
              }
              ++n;
            }
            continue;
          }
          const int q0 = lq;
          ++lq;
          while (lq < lxe && mhas(m, lq + 8 * ly + 64 * lz) &&
                 ((bits[a + (lq - q0)] >> s) & 1ull))
            ++lq;
          if (WRITE) {
            const uint32_t src = (uint32_t)(loff + pos[a]);
            const uint32_t dst =
                (uint32_t)((bx * 8 + q0 - T.ox) + T.pad[0] * (y - T.oy) + T.pad[1] * (z - T.oz));
            runs[out + n] = pack_run(src, dst, (uint32_t)(lq - q0));
          }
          ++n;
        }
      }
      x = xend;
    }
    if (!WRITE) rowcnt[gi] = n;
  }
}

__global__ void k_set_ranges(int n, TileHdr* sub, const int64_t* rowbase, const int64_t* runstart,
                             int64_t roff) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  sub[q].r0 = (int32_t)(roff + runstart[rowbase[q]]);
  sub[q].r1 = (int32_t)(roff + runstart[rowbase[q + 1]]);
}

// ---------------------------------------------------------------- apply kernels
// x_i = (R_j r) for every member i of the concatenated subdomains: gidx < nown
// indexes the owned vector, larger values the received halo (distributed RAS).
__global__ void k_gather(int64_t n, const int64_t* gidx, const double* r, const double* rh,
                         int64_t nown, double* x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = gidx[i];
    x[i] = g < 0 ? 0.0 : (g < nown ? r[g] : rh[g - nown]);  // g < 0: a segment's pad entry
  }
}

// one thread per segment
__global__ void k_inner_init(InnerState* st, int S, int k) {
  const int s = threadIdx.x;
  if (s >= S) return;
  InnerState& q = st[s];
  const double beta = sqrt(q.beta2);
  q.g[0] = beta;
  for (int i = 1; i <= k; ++i) q.g[i] = 0.0;
  q.sc[0] = beta > 0.0 ? 1.0 / beta : 0.0;
  q.kk = beta > 0.0 ? k : 0;
}

// Delayed-CGS2 step j of one segment's inner GMRES, the arithmetic of krylov.cu
// dcgs_step_body without a convergence test: finalise column j-1 ([cpend + b;
// rho], Givens), then the coefficients of the update pass.  Run by the block (nt = blockDim.x <= 256 threads) of the segmented reduction
// pass that completes segment s (InnerStepEpi): the inner solves are rank-local,
// so no reduction sits between the pass and the step.
__device__ void inner_step_body(InnerState& q, int j) {
  constexpr int ld = kMaxInner + 1, ldc = kMaxInner + 2;
  const int k = j + 1, tid = threadIdx.x, nt = blockDim.x;
  const double* b = q.red;
  const double* d = q.red + k;
  __shared__ double sbb[8], sbd[8];
  __shared__ int sstop;
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
  const double alpha = q.red[j], gamma = q.red[k + j];
  const double rho2 = alpha - bb;
  const bool brk = !(rho2 > 1e-28 * alpha);
  const double rho = brk ? 1.0 : sqrt(rho2);  // broken: the segment stops at kk = j
  if (j >= 1)
    for (int i = tid; i < j; i += nt) q.Hr[(size_t)(j - 1) * ld + i] = q.cpend[i] + b[i];
  __syncthreads();
  if (tid == 0) {
    sstop = 0;
    if (j == 0) {
      q.g[0] *= brk ? 0.0 : rho;  // u_0 = r_j / beta: r_j = (beta rho) q_0
      if (brk) q.kk = 0;
    } else if (q.kk >= j) {
      double* Hr = q.Hr + (size_t)(j - 1) * ld;
      double* H = q.H + (size_t)(j - 1) * ld;
      Hr[j] = brk ? 0.0 : rho;
      for (int i = 0; i <= j; ++i) H[i] = Hr[i];
      const int c = j - 1;
      for (int i = 0; i < c; ++i) {
        const double t = q.cs[i] * H[i] + q.sn[i] * H[i + 1];
        H[i + 1] = -q.sn[i] * H[i] + q.cs[i] * H[i + 1];
        H[i] = t;
      }
      const double den = hypot(H[c], H[c + 1]);
      if (den == 0.0) {
        q.cs[c] = 1.0;
        q.sn[c] = 0.0;
      } else {
        q.cs[c] = H[c] / den;
        q.sn[c] = H[c + 1] / den;
      }
      H[c] = q.cs[c] * H[c] + q.sn[c] * H[c + 1];
      H[c + 1] = 0.0;
      q.g[c + 1] = -q.sn[c] * q.g[c];
      q.g[c] = q.cs[c] * q.g[c];
      if (brk && q.kk > j) q.kk = j;  // happy breakdown: solution in the first j columns
    }
    if (brk) sstop = 1;
  }
  __syncthreads();
  double* cb = q.coef;
  double* ce = q.coef + ldc;
  if (sstop) {  // harmless coefficients for the (unused) rest of this segment
    for (int i = tid; i < j; i += nt) cb[i] = ce[i] = 0.0;
    if (tid == 0) {
      q.coef[2 * ldc] = 1.0;
      q.coef[2 * ldc + 1] = 0.0;
    }
    return;
  }
  const double mu = (gamma - bd) / rho2;
  for (int l = tid; l <= j; l += nt) {
    double gl = 0.0;  // (Hr b)_l
    for (int i = (l > 0 ? l - 1 : 0); i < j; ++i) gl += q.Hr[(size_t)i * ld + l] * b[i];
    const double ql = l < j ? d[l] : rho * mu;
    q.cpend[l] = (ql - gl) / rho;
  }
  for (int i = tid; i < j; i += nt) {
    cb[i] = b[i];
    ce[i] = d[i] - mu * b[i];
  }
  if (tid == 0) {
    q.coef[2 * ldc] = rho;
    q.coef[2 * ldc + 1] = mu;
  }
}
struct InnerStepEpi {
  InnerState* st;
  int j;
  __device__ void operator()(int s) const { inner_step_body(st[s], j); }
};

__global__ void k_inner_lsq(InnerState* st) {
  InnerState& q = st[blockIdx.x];
  constexpr int ld = kMaxInner + 1;
  const int k = q.kk;
  const int lane = threadIdx.x;
  for (int i = k - 1; i >= 0; --i) {
    double s = 0.0;
    for (int p = i + 1 + lane; p < k; p += 32) s += q.H[(size_t)p * ld + i] * q.y[p];
    s = vec::warp_sum(s);
    if (lane == 0) q.y[i] = (q.g[i] - s) / q.H[(size_t)i * ld + i];
    __syncwarp();
    __threadfence_block();
  }
}

// ---------------------------------------------------------------- host helpers
struct DBuf {
  void* p = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const {
    return (T*)p;
  }
  int alloc(size_t bytes) {
    if (p) cudaFree(p);
    p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(bytes, 16)) != cudaSuccess)
      return fail(CPM_ERR_NOMEM, "cpm_ras_setup: device allocation failed");
    return CPM_OK;
  }
};

template <class T>
int scan(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  CPM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  DBuf tb;
  CPM_TRY(tb.alloc(tmp));
  CPM_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, tmp, in, out, n, s));
  return CPM_OK;
}

template <class T>
int read1(const T* d, T* h, cudaStream_t s) {
  CPM_CUDA(cudaMemcpyAsync(h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  return CPM_OK;
}

inline int g1(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

struct RasImpl {
  cpm_band mb;            // the multi-band (owns=false): sub-tiles, runs, local acell, vb
  int S = 0, k = 0;
  int64_t ntot = 0;                 // concatenated segments, pads included
  int64_t nmem = 0;                 // members (without the pads)
  int aligned = 0;                  // segment starts are multiples of 32 elements
  std::vector<int64_t> off_h;  // S + 1
  int64_t* off = nullptr;      // device S + 1
  int64_t* gidx = nullptr;     // Ntot
  int64_t *lo = nullptr, *hi = nullptr, *xoff = nullptr;  // disjoint local ranges
  double* V = nullptr;         // (k+1) * ldv
  int64_t ldv = 0;
  double* W = nullptr;
  double* partial = nullptr;
  InnerState* st = nullptr;
  unsigned* counters = nullptr;
  int gps = 1;
  // distributed RAS (a rank's subdomains of a partitioned band)
  int rank = 0, nranks = 1, sub0 = 0, nsubGlobal = 0;
  int64_t ownLo = 0, nOwned = 0, nHalo = 0, nSend = 0;
  std::vector<int64_t> halo_h;                       // received global indices (sorted)
  double* hbuf = nullptr;                            // received values
  double* zeros = nullptr;                           // the fill runs' zero source (16 doubles)
  int64_t* sendidx = nullptr;                        // owned local indices to send
  double* sendbuf = nullptr;
  std::vector<int64_t> sendCount, sendOff, recvCount, recvOff;
  ~RasImpl() {
    void* ps[] = {off, gidx, lo, hi, xoff, V, W, partial, st, counters, hbuf, sendidx, sendbuf, zeros};
    for (void* p : ps)
      if (p) cudaFree(p);
    void* mp[] = {mb.tiles, mb.runs, mb.vb, mb.acell};
    for (void* p : mp)
      if (p) cudaFree(p);
  }
};

// sub0, nsl: this rank's subdomains [sub0, sub0 + nsl) of S; own_lo, nown: its owned
// band-order range (the whole band on one GPU); nranks: for the halo owners.
int ras_setup_device(const cpm_band* B, int S, int overlap, int k, double c, cudaStream_t s,
                     cpm_ras** out, int sub0, int nsl, int64_t own_lo, int64_t nown, int rank,
                     int nranks) {
  if (!B || !out) return fail(CPM_ERR_ARG, "cpm_ras_setup: null argument");
  *out = nullptr;
  if (S < 1 || S > 64) return fail(CPM_ERR_ARG, "cpm_ras_setup: n_sub must be in [1, 64]");
  if (overlap < 0 || overlap > 64) return fail(CPM_ERR_ARG, "cpm_ras_setup: overlap must be in [0, 64]");
  if (k < 1 || k > kMaxInner) return fail(CPM_ERR_ARG, "cpm_ras_setup: k_inner must be in [1, 64]");
  if (!B->owns || B->nA < S) return fail(CPM_ERR_ARG, "cpm_ras_setup: needs a full band with n_active >= n_sub");
  const int64_t nA = B->nA;
  const int nT = B->nT;
  if (sub0 < 0 || nsl < 1 || sub0 + nsl > S) return fail(CPM_ERR_ARG, "cpm_ras_setup: bad subdomain range");
  auto R = std::make_unique<RasImpl>();
  R->S = nsl;  // segments of the batched inner solves: this rank's subdomains
  R->k = k;
  R->rank = rank;
  R->nranks = nranks;
  R->sub0 = sub0;
  R->nsubGlobal = S;
  R->ownLo = own_lo;
  R->nOwned = nown;

  // neighbour table and membership bits
  DBuf nbr, bits0, bits1;
  CPM_TRY(nbr.alloc(sizeof(int) * 6 * (size_t)nA));
  CPM_TRY(bits0.alloc(sizeof(uint64_t) * (size_t)nA));
  CPM_TRY(bits1.alloc(sizeof(uint64_t) * (size_t)nA));
  k_nbr_active<<<nT, 256, 0, s>>>(B->tiles, B->amask, B->acell, nbr.as<int>());
  count_launch();
  k_member_init<<<g1(nA), 256, 0, s>>>(nA, S, bits0.as<uint64_t>());
  count_launch();
  uint64_t* bits = bits0.as<uint64_t>();
  uint64_t* other = bits1.as<uint64_t>();
  for (int l = 0; l < overlap; ++l) {
    k_member_grow<<<g1(nA), 256, 0, s>>>(nA, nbr.as<int>(), bits, other);
    count_launch();
    std::swap(bits, other);
  }
  CPM_CUDA(cudaGetLastError());

  // phase A: sizes
  DBuf flag, pos, has, inc, incpos;
  CPM_TRY(flag.alloc(sizeof(int) * (size_t)(nA + 1)));
  CPM_TRY(pos.alloc(sizeof(int) * (size_t)(nA + 1)));
  CPM_TRY(has.alloc(sizeof(int) * (size_t)(nT + 1)));
  CPM_TRY(inc.alloc(sizeof(int) * (size_t)(nT + 1)));
  CPM_TRY(incpos.alloc(sizeof(int) * (size_t)(nT + 1)));
  std::vector<int64_t> nloc(nsl), ntl(nsl);
  auto member_scan = [&](int sd) -> int {
    k_flag_bit<<<g1(nA + 1), 256, 0, s>>>(nA, bits, sd, flag.as<int>());
    count_launch();
    CPM_TRY(scan(flag.as<int>(), pos.as<int>(), nA + 1, s));
    k_tile_has<<<nT, 256, 0, s>>>(B->tiles, bits, sd, has.as<int>());
    count_launch();
    k_tile_include<<<(nT + 256) / 256, 256, 0, s>>>(nT, B->tiles, has.as<int>(), inc.as<int>());
    count_launch();
    CPM_TRY(scan(inc.as<int>(), incpos.as<int>(), nT + 1, s));
    CPM_CUDA(cudaGetLastError());
    return CPM_OK;
  };
  for (int ls = 0; ls < nsl; ++ls) {
    CPM_TRY(member_scan(sub0 + ls));
    int nl = 0, nt = 0;
    CPM_TRY(read1(pos.as<int>() + nA, &nl, s));
    CPM_TRY(read1(incpos.as<int>() + nT, &nt, s));
    nloc[ls] = nl;
    ntl[ls] = nt;
  }
  // segments start at multiples of 32 elements (256 B): the inner Krylov reduction
  // pass then runs the register-direct kernel with 16-byte loads (vecops.cuh); the
  // pad entries of a segment are zero in every inner vector (gidx -1, the apply never
  // writes them) and add nothing to its dot products.  CPM_RAS_ALIGN=0: unpadded.
  static const bool align = !(getenv("CPM_RAS_ALIGN") && *getenv("CPM_RAS_ALIGN") == '0');
  const int64_t seg_align = align ? 32 : 1;
  R->off_h.assign(nsl + 1, 0);
  std::vector<int64_t> toff(nsl + 1, 0);
  R->nmem = 0;
  for (int ls = 0; ls < nsl; ++ls) {
    R->off_h[ls + 1] = R->off_h[ls] + (nloc[ls] + seg_align - 1) / seg_align * seg_align;
    toff[ls + 1] = toff[ls] + ntl[ls];
    R->nmem += nloc[ls];
  }
  R->ntot = R->off_h[nsl];
  R->aligned = align ? 1 : 0;
  const int nTs = (int)toff[nsl];
  if (R->ntot >= INT32_MAX) return fail(CPM_ERR_LIMIT, "cpm_ras_setup: concatenated subdomains too large");

  cpm_band& M = R->mb;
  M.surf = B->surf;
  M.h = B->h;
  M.lam = B->lam;
  M.L = B->L;
  M.M = B->M;
  M.owns = false;
  M.nA = R->ntot;
  M.nE = B->nE;
  M.nT = nTs;
  M.maxBox = B->maxBox;
  // cells of Sigma_A outside a subdomain are filled from a zero buffer (fill runs with
  // source index ntot = srcSplit); CPM_RAS_ZRUNS=0: cleared boxes instead (zeroFill)
  static const bool zruns = !(getenv("CPM_RAS_ZRUNS") && *getenv("CPM_RAS_ZRUNS") == '0');
  const int64_t zsrc = zruns ? R->ntot : -1;
  M.zeroFill = !zruns;
  M.srcSplit = zruns ? (uint32_t)R->ntot : 0xffffffffu;
  CPM_CUDA(cudaMalloc(&R->zeros, sizeof(double) * 16));
  CPM_CUDA(cudaMemsetAsync(R->zeros, 0, sizeof(double) * 16, s));
  M.tx = B->tx;
  M.ty = B->ty;
  M.tz = B->tz;
  M.eoff = B->eoff;
  M.rnd = B->rnd;
  M.itemOrder = B->itemOrder;
  CPM_CUDA(cudaMalloc(&M.tiles, sizeof(TileHdr) * std::max(nTs, 1)));
  CPM_CUDA(cudaMalloc(&M.acell, sizeof(uint16_t) * std::max<int64_t>(R->ntot, 1)));
  CPM_CUDA(cudaMalloc(&M.vb, sizeof(double) * kBrickCells * (size_t)std::max(nTs, 1)));
  CPM_CUDA(cudaMemsetAsync(M.vb, 0, sizeof(double) * kBrickCells * (size_t)std::max(nTs, 1), s));
  CPM_CUDA(cudaMalloc(&R->gidx, sizeof(int64_t) * std::max<int64_t>(R->ntot, 1)));
  CPM_CUDA(cudaMemsetAsync(R->gidx, 0xff, sizeof(int64_t) * std::max<int64_t>(R->ntot, 1), s));  // pads: -1

  // phase B: per-subdomain structures
  DBuf tmap;
  CPM_TRY(tmap.alloc(sizeof(int) * (size_t)nT));
  std::vector<DBuf> runbuf(nsl);
  std::vector<int64_t> nrun(nsl, 0);
  std::vector<int64_t> lo_h(nsl), hi_h(nsl), xo_h(nsl);
  DBuf dblo, dbdim;
  CPM_TRY(dblo.alloc(3 * sizeof(int)));
  CPM_TRY(dbdim.alloc(3 * sizeof(int)));
  CPM_CUDA(cudaMemcpyAsync(dblo.p, B->blo, 3 * sizeof(int), cudaMemcpyHostToDevice, s));
  CPM_CUDA(cudaMemcpyAsync(dbdim.p, B->bdim, 3 * sizeof(int), cudaMemcpyHostToDevice, s));
  for (int ls = 0; ls < nsl; ++ls) {
    const int sd = sub0 + ls;  // global subdomain (membership bit), ls its segment here
    CPM_TRY(member_scan(sd));
    const int64_t loff = R->off_h[ls];
    const int to = (int)toff[ls], nt = (int)ntl[ls];
    k_subtiles<<<(nT + 255) / 256, 256, 0, s>>>(nT, B->tiles, inc.as<int>(), incpos.as<int>(),
                                                 pos.as<int>(), loff, to, ls, M.tiles, tmap.as<int>());
    count_launch();
    if (nt > 0) {
      k_subtile_nbrs<<<(nt + 255) / 256, 256, 0, s>>>(nt, M.tiles + to, tmap.as<int>());
      count_launch();
    }
    k_local_index<<<g1(nA), 256, 0, s>>>(nA, flag.as<int>(), pos.as<int>(), loff, B->acell, R->gidx,
                                         M.acell);
    count_launch();
    // disjoint (slab) range in local numbering
    const int64_t d0 = slab_lo(sd, nA, S), d1 = slab_lo(sd + 1, nA, S);
    int ld0 = 0;
    CPM_TRY(read1(pos.as<int>() + d0, &ld0, s));
    lo_h[ls] = ld0;
    hi_h[ls] = ld0 + (d1 - d0);
    xo_h[ls] = d0 - own_lo;  // the disjoint slab lies in this rank's owned range
    // runs
    if (nt > 0) {
      DBuf nrows, rowbase, rowcnt, runstart;
      CPM_TRY(nrows.alloc(sizeof(int64_t) * (nt + 1)));
      CPM_TRY(rowbase.alloc(sizeof(int64_t) * (nt + 1)));
      k_rows<<<(nt + 256) / 256, 256, 0, s>>>(nt, M.tiles + to, nrows.as<int64_t>());
      count_launch();
      CPM_TRY(scan(nrows.as<int64_t>(), rowbase.as<int64_t>(), nt + 1, s));
      int64_t rows = 0;
      CPM_TRY(read1(rowbase.as<int64_t>() + nt, &rows, s));
      CPM_TRY(rowcnt.alloc(sizeof(int64_t) * (rows + 1)));
      CPM_TRY(runstart.alloc(sizeof(int64_t) * (rows + 1)));
      CPM_CUDA(cudaMemsetAsync(rowcnt.p, 0, sizeof(int64_t) * (rows + 1), s));
      k_sub_runs<false><<<nt, 128, 0, s>>>(M.tiles + to, B->tiles, B->amask, B->bmap, dblo.as<int>(),
                                           dbdim.as<int>(), bits, sd, pos.as<int>(), loff,
                                           rowbase.as<int64_t>(), rowcnt.as<int64_t>(), nullptr,
                                           nullptr, zsrc);
      count_launch();
      CPM_TRY(scan(rowcnt.as<int64_t>(), runstart.as<int64_t>(), rows + 1, s));
      int64_t nr = 0;
      CPM_TRY(read1(runstart.as<int64_t>() + rows, &nr, s));
      CPM_TRY(runbuf[ls].alloc(sizeof(uint64_t) * (size_t)nr));
      k_sub_runs<true><<<nt, 128, 0, s>>>(M.tiles + to, B->tiles, B->amask, B->bmap, dblo.as<int>(),
                                          dbdim.as<int>(), bits, sd, pos.as<int>(), loff,
                                          rowbase.as<int64_t>(), rowcnt.as<int64_t>(),
                                          runstart.as<int64_t>(), runbuf[ls].as<uint64_t>(), zsrc);
      count_launch();
      int64_t roff = 0;
      for (int q = 0; q < ls; ++q) roff += nrun[q];
      k_set_ranges<<<(nt + 255) / 256, 256, 0, s>>>(nt, M.tiles + to, rowbase.as<int64_t>(),
                                                     runstart.as<int64_t>(), roff);
      count_launch();
      nrun[ls] = nr;
      CPM_CUDA(cudaStreamSynchronize(s));
    }
    CPM_CUDA(cudaGetLastError());
  }
  int64_t totRuns = 0;
  for (int ls = 0; ls < nsl; ++ls) totRuns += nrun[ls];
  if (totRuns >= (int64_t)INT32_MAX) return fail(CPM_ERR_LIMIT, "cpm_ras_setup: too many runs");
  CPM_CUDA(cudaMalloc(&M.runs, sizeof(uint64_t) * std::max<int64_t>(totRuns, 1)));
  for (int ls = 0, ro = 0; ls < nsl; ro += (int)nrun[ls], ++ls)
    if (nrun[ls] > 0)
      CPM_CUDA(cudaMemcpyAsync(M.runs + ro, runbuf[ls].p, sizeof(uint64_t) * nrun[ls],
                               cudaMemcpyDeviceToDevice, s));
  M.nRuns = totRuns;

  // members outside the owned range come from other ranks (the RAS halo): gidx
  // becomes an index into [owned | halo]
  if (own_lo != 0 || nown != nA) {
    std::vector<int64_t> g(R->ntot);
    if (R->ntot > 0)
      CPM_CUDA(cudaMemcpy(g.data(), R->gidx, sizeof(int64_t) * R->ntot, cudaMemcpyDeviceToHost));
    std::vector<int64_t>& H = R->halo_h;
    for (int64_t v : g)
      if (v >= 0 && (v < own_lo || v >= own_lo + nown)) H.push_back(v);
    std::sort(H.begin(), H.end());
    H.erase(std::unique(H.begin(), H.end()), H.end());
    for (int64_t& v : g)
      if (v >= 0)
        v = (v >= own_lo && v < own_lo + nown) ? v - own_lo
                                               : nown + (std::lower_bound(H.begin(), H.end(), v) - H.begin());
    if (R->ntot > 0)
      CPM_CUDA(cudaMemcpy(R->gidx, g.data(), sizeof(int64_t) * R->ntot, cudaMemcpyHostToDevice));
    R->nHalo = (int64_t)H.size();
    CPM_CUDA(cudaMalloc(&R->hbuf, sizeof(double) * std::max<int64_t>(R->nHalo, 1)));
    // receive plan: the halo is sorted, hence grouped by owner (slab bounds, reading R8)
    R->recvCount.assign(nranks, 0);
    R->recvOff.assign(nranks + 1, 0);
    for (int64_t v : H) {
      int q = (int)((v * nranks) / nA);
      while (q + 1 < nranks && v >= slab_lo(q + 1, nA, nranks)) ++q;
      while (q > 0 && v < slab_lo(q, nA, nranks)) --q;
      R->recvCount[q]++;
    }
    for (int q = 0; q < nranks; ++q) R->recvOff[q + 1] = R->recvOff[q] + R->recvCount[q];
    if (R->recvCount[rank] != 0) return fail(CPM_ERR_GEOM, "cpm_part_ras_setup: halo contains owned nodes");
  }

  // segment tables and inner workspace
  CPM_CUDA(cudaMalloc(&R->off, sizeof(int64_t) * (nsl + 1)));
  CPM_CUDA(cudaMalloc(&R->lo, sizeof(int64_t) * nsl));
  CPM_CUDA(cudaMalloc(&R->hi, sizeof(int64_t) * nsl));
  CPM_CUDA(cudaMalloc(&R->xoff, sizeof(int64_t) * nsl));
  CPM_CUDA(cudaMemcpyAsync(R->off, R->off_h.data(), sizeof(int64_t) * (nsl + 1), cudaMemcpyHostToDevice, s));
  CPM_CUDA(cudaMemcpyAsync(R->lo, lo_h.data(), sizeof(int64_t) * nsl, cudaMemcpyHostToDevice, s));
  CPM_CUDA(cudaMemcpyAsync(R->hi, hi_h.data(), sizeof(int64_t) * nsl, cudaMemcpyHostToDevice, s));
  CPM_CUDA(cudaMemcpyAsync(R->xoff, xo_h.data(), sizeof(int64_t) * nsl, cudaMemcpyHostToDevice, s));
  R->ldv = (R->ntot + 63) / 64 * 64;
  CPM_CUDA(cudaMalloc(&R->V, sizeof(double) * (size_t)R->ldv * (k + 1)));
  CPM_CUDA(cudaMalloc(&R->W, sizeof(double) * (size_t)R->ldv));
  CPM_CUDA(cudaMemsetAsync(R->W, 0, sizeof(double) * (size_t)R->ldv, s));  // pad entries stay 0
  int64_t maxn = 0;
  for (int ls = 0; ls < nsl; ++ls) maxn = std::max(maxn, nloc[ls]);
  // blocks per segment of the inner Krylov passes; CPM_RAS_GPS overrides (experiment)
  const int gcap = getenv("CPM_RAS_GPS") ? std::max(1, atoi(getenv("CPM_RAS_GPS"))) : std::max(1, kMaxBlocks / nsl / 2);
  R->gps = (int)std::max<int64_t>(1, std::min<int64_t>((maxn + 255) / 256, gcap));
  CPM_CUDA(cudaMalloc(&R->partial, sizeof(double) * (size_t)nsl * R->gps * (2 * (kMaxInner + 2) + 8)));
  CPM_CUDA(cudaMalloc(&R->st, sizeof(InnerState) * nsl));
  CPM_CUDA(cudaMemsetAsync(R->st, 0, sizeof(InnerState) * nsl, s));
  CPM_CUDA(cudaMalloc(&R->counters, sizeof(unsigned) * nsl * 4));
  CPM_CUDA(cudaMemsetAsync(R->counters, 0, sizeof(unsigned) * nsl * 4, s));
  CPM_CUDA(cudaStreamSynchronize(s));

  cpm_ras* ras = new cpm_ras();
  ras->band = B;
  ras->nsub = S;
  ras->overlap = overlap;
  ras->k = k;
  ras->c = c;
  ras->impl = R.release();
  *out = ras;
  return CPM_OK;
}

int ras_apply_device(const cpm_ras* ras, const double* r, double* z, cudaStream_t s,
                     const double* r_halo) {
  RasImpl* R = (RasImpl*)ras->impl;
  if (!r_halo) r_halo = R->hbuf;
  const int S = R->S, k = R->k;
  vec::Seg Sg{R->off, S, R->gps};
  Sg.aligned = R->aligned;
  const int grid = S * R->gps;
  constexpr int lds = (int)(sizeof(InnerState) / sizeof(double));  // stride between segments' states
  InnerState* st = R->st;
  double* base = (double*)st;
  // member offsets inside InnerState, in doubles
  const int o_beta2 = (int)(offsetof(InnerState, beta2) / sizeof(double));
  const int o_sc = (int)(offsetof(InnerState, sc) / sizeof(double));
  const int o_y = (int)(offsetof(InnerState, y) / sizeof(double));
  {
    ProfScope ps(K_OTHER, s);
    k_gather<<<g1(R->ntot), 256, 0, s>>>(R->ntot, R->gidx, r, r_halo, R->nOwned, R->V);
    count_launch();
    vec::k_sub_nrm2<<<grid, VB, 0, s>>>(Sg, R->V, nullptr, nullptr, R->partial, base + o_beta2, lds,
                                        R->counters);
    count_launch();
    k_inner_init<<<1, 64, 0, s>>>(st, S, k);
    count_launch();
  }
  const int o_red = (int)(offsetof(InnerState, red) / sizeof(double));
  const int o_coef = (int)(offsetof(InnerState, coef) / sizeof(double));
  {  // V_0 = R_j r / beta_j: the first lagged vector of every segment
    ProfScope ps(K_AXPY, s);
    vec::k_scale<<<grid, VB, 0, s>>>(Sg, R->V, base + o_sc, lds, 0, R->V);
    count_launch();
  }
  // delayed CGS2 (krylov.cu): per inner step one apply, one reduction pass, one
  // update pass; step k only finalises the last Hessenberg column
  for (int j = 0; j <= k; ++j) {
    if (j < k)
      CPM_TRY(apply_device_split(&R->mb, ras->c, R->V + (size_t)j * R->ldv, R->zeros, R->W, nullptr, 0, s));
    {  // the block that completes segment s's reduction runs its step (epilogue)
      ProfScope ps(K_MDOT, s);
      CPM_TRY(launch_dcgs_dots_epi(Sg, j + 1, R->V, R->ldv, R->W, R->partial, 2 * (kMaxInner + 2) + 8,
                                   base + o_red, lds, R->counters + S, s, nullptr,
                                   InnerStepEpi{st, j}));
    }
    if (j < k) {
      ProfScope ps(K_CGS_UPDATE, s);
      CPM_TRY(launch_dcgs_update(Sg, j + 1, R->V, R->ldv, R->W, base + o_coef, kMaxInner + 2, lds, s));
    }
  }
  {
    ProfScope ps(K_AXPY, s);
    k_inner_lsq<<<S, 32, 0, s>>>(st);
    count_launch();
    const int* kks = (const int*)((const char*)st + offsetof(InnerState, kk));
    vec::k_combine<<<grid, VB, 0, s>>>(Sg, R->V, R->ldv, base + o_y, lds, nullptr, 0, kks,
                                       (int)(sizeof(InnerState) / sizeof(int)), 0, R->lo, R->hi,
                                       R->xoff, z, 0);
    count_launch();
  }
  CPM_CUDA(cudaGetLastError());
  return CPM_OK;
}

int ras_exchange(const cpm_ras* ras, const cpm_comm* comm, const double* r_owned, cudaStream_t s) {
  const RasImpl* R = (const RasImpl*)ras->impl;
  if (R->nranks == 1) return CPM_OK;
  return halo_exchange(comm, R->rank, R->nranks, r_owned, R->nSend, R->sendidx, R->sendbuf,
                       R->sendCount, R->sendOff, R->hbuf, R->recvCount, R->recvOff, s);
}

}  // namespace cpm

using namespace cpm;
extern "C" {
int cpm_ras_setup(const cpm_band* band, int n_sub, int overlap, int k_inner, double c, void* stream,
                  cpm_ras** out) {
  if (!band) return fail(CPM_ERR_ARG, "cpm_ras_setup: null argument");
  return ras_setup_device(band, n_sub, overlap, k_inner, c, (cudaStream_t)stream, out, 0, n_sub, 0,
                          band->nA, 0, 1);
}

int cpm_part_ras_setup(const cpm_part* part, int n_sub, int overlap, int k_inner, double c,
                       void* stream, cpm_ras** out) {
  if (!part || !out) return fail(CPM_ERR_ARG, "cpm_part_ras_setup: null argument");
  const int R = part->nranks;
  if (n_sub < R || n_sub % R != 0)
    return fail(CPM_ERR_ARG, "cpm_part_ras_setup: n_sub must be a multiple of the number of ranks "
                             "(PAPER.md:213)");
  const int per = n_sub / R;
  return ras_setup_device(part->band, n_sub, overlap, k_inner, c, (cudaStream_t)stream, out,
                          part->rank * per, per, part->lo, part->nOwned, part->rank, R);
}

int cpm_ras_get_info(const cpm_ras* ras, cpm_ras_info* info) {
  if (!ras || !info) return fail(CPM_ERR_ARG, "cpm_ras_get_info: null argument");
  const RasImpl* R = (const RasImpl*)ras->impl;
  memset(info, 0, sizeof(*info));
  info->n_sub = R->nsubGlobal;
  info->sub0 = R->sub0;
  info->n_sub_local = R->S;
  info->rank = R->rank;
  info->nranks = R->nranks;
  info->n_members = R->nmem;
  info->n_owned = R->nOwned;
  info->n_halo = R->nHalo;
  info->n_send = R->nSend;
  return CPM_OK;
}

int cpm_ras_halo_nodes(const cpm_ras* ras, int64_t* halo_host) {
  if (!ras) return fail(CPM_ERR_ARG, "cpm_ras_halo_nodes: null argument");
  const RasImpl* R = (const RasImpl*)ras->impl;
  if (R->nHalo > 0 && !halo_host) return fail(CPM_ERR_ARG, "cpm_ras_halo_nodes: null output");
  if (R->nHalo > 0) memcpy(halo_host, R->halo_h.data(), sizeof(int64_t) * R->nHalo);
  return CPM_OK;
}

int cpm_ras_set_send(cpm_ras* ras, const int64_t* send_global, const int64_t* counts) {
  if (!ras || !counts) return fail(CPM_ERR_ARG, "cpm_ras_set_send: null argument");
  RasImpl* R = (RasImpl*)ras->impl;
  const int nr = R->nranks;
  R->sendCount.assign(counts, counts + nr);
  R->sendOff.assign(nr + 1, 0);
  for (int q = 0; q < nr; ++q) {
    if (counts[q] < 0) return fail(CPM_ERR_ARG, "cpm_ras_set_send: negative count");
    R->sendOff[q + 1] = R->sendOff[q] + counts[q];
  }
  const int64_t n = R->sendOff[nr];
  if (n > 0 && !send_global) return fail(CPM_ERR_ARG, "cpm_ras_set_send: null index list");
  std::vector<int64_t> loc(n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t a = send_global[i];
    if (a < R->ownLo || a >= R->ownLo + R->nOwned)
      return fail(CPM_ERR_ARG, "cpm_ras_set_send: requested node not owned");
    loc[i] = a - R->ownLo;
  }
  if (R->sendidx) cudaFree(R->sendidx);
  if (R->sendbuf) cudaFree(R->sendbuf);
  R->sendidx = nullptr;
  R->sendbuf = nullptr;
  CPM_CUDA(cudaMalloc(&R->sendidx, sizeof(int64_t) * std::max<int64_t>(n, 1)));
  CPM_CUDA(cudaMalloc(&R->sendbuf, sizeof(double) * std::max<int64_t>(n, 1)));
  if (n > 0) CPM_CUDA(cudaMemcpy(R->sendidx, loc.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice));
  R->nSend = n;
  return CPM_OK;
}

int cpm_part_ras_apply_local(const cpm_ras* ras, const double* r_owned, const double* r_halo,
                             double* z_owned, void* stream) {
  if (!ras || !r_owned || !z_owned) return fail(CPM_ERR_ARG, "cpm_part_ras_apply_local: null argument");
  const RasImpl* R = (const RasImpl*)ras->impl;
  if (R->nHalo > 0 && !r_halo) return fail(CPM_ERR_ARG, "cpm_part_ras_apply_local: null halo");
  if (!is_device_ptr(r_owned) || !is_device_ptr(z_owned) || (r_halo && !is_device_ptr(r_halo)))
    return fail(CPM_ERR_ARG, "cpm_part_ras_apply_local: vectors must be device memory");
  return ras_apply_device(ras, r_owned, z_owned, (cudaStream_t)stream, r_halo ? r_halo : R->hbuf);
}

int cpm_part_ras_apply(const cpm_ras* ras, const cpm_comm* comm, const double* r_owned,
                       double* z_owned, void* stream) {
  if (!ras || !r_owned || !z_owned) return fail(CPM_ERR_ARG, "cpm_part_ras_apply: null argument");
  if (!is_device_ptr(r_owned) || !is_device_ptr(z_owned))
    return fail(CPM_ERR_ARG, "cpm_part_ras_apply: vectors must be device memory");
  cudaStream_t s = (cudaStream_t)stream;
  CPM_TRY(ras_exchange(ras, comm, r_owned, s));
  return ras_apply_device(ras, r_owned, z_owned, s);
}

int cpm_ras_apply(const cpm_ras* ras, const double* r, double* z, void* stream) {
  if (!ras || !r || !z) return fail(CPM_ERR_ARG, "cpm_ras_apply: null argument");
  if (((const RasImpl*)ras->impl)->nOwned != ras->band->nA)
    return fail(CPM_ERR_ARG, "cpm_ras_apply: partitioned preconditioner (use cpm_part_ras_apply)");
  if ((const void*)r == (const void*)z) return fail(CPM_ERR_ARG, "cpm_ras_apply: r and z must not alias");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = ras->band->nA;
  const bool dr = is_device_ptr(r), dz = is_device_ptr(z);
  if (dr && dz) return ras_apply_device(ras, r, z, s);
  double *br = nullptr, *bz = nullptr;
  CPM_CUDA(cudaMalloc(&br, sizeof(double) * n));
  if (cudaMalloc(&bz, sizeof(double) * n) != cudaSuccess) {
    cudaFree(br);
    return fail(CPM_ERR_NOMEM, "cpm_ras_apply: staging allocation failed");
  }
  int rc = CPM_OK;
  if (cudaMemcpyAsync(br, r, sizeof(double) * n, dr ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s) != cudaSuccess)
    rc = fail(CPM_ERR_CUDA, "cpm_ras_apply: copy failed");
  if (rc == CPM_OK) rc = ras_apply_device(ras, br, bz, s);
  if (rc == CPM_OK && cudaMemcpyAsync(z, bz, sizeof(double) * n, dz ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s) != cudaSuccess)
    rc = fail(CPM_ERR_CUDA, "cpm_ras_apply: copy-back failed");
  cudaStreamSynchronize(s);
  cudaFree(br);
  cudaFree(bz);
  return rc;
}

void cpm_ras_free(cpm_ras* r) {
  if (!r) return;
  delete (RasImpl*)r->impl;
  delete r;
}
}
