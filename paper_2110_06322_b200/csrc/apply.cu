// apply.cu — matrix-free stabilised CPM operator (north_star item 2).
//
//   y = c u - [Delta_h E u - (6/h^2)(u - E u)]          (Eq. 4, d = 3)
//     = (c + 6/h^2) u - (1/h^2) sum_{6 nbrs j} (E u)_j    (the centre (E u)_i terms cancel)
//
// Two kernels per apply:
//   k_extend_nt (one CTA of 128 threads per tile = occupied 8^3 brick, up to 4
//             eval nodes per thread): stage the cells of u the tile's stencils read
//             into a shared-memory box (fill runs of consecutive band-order sources,
//             8 lanes per run, cp.async); for every eval node (Sigma_A u Sigma_G in
//             the brick) recompute the tricubic Lagrange weights from its fractional
//             offsets and contract x, then y, then z.  A tile's nodes
//             are ordered (build time) so adjacent lane pairs read one address and
//             the 16 pair addresses of a warp distinct banks.  E u goes to
//             vb[tile * 512 + cell].
//   k_laplace (one CTA of 128 threads per tile): gather the tile's E u and the face
//             layers of its 6 neighbour tiles into a dense 10^3 halo brick in shared
//             memory, then the 7-point combination for every output node.
// Both kernels bulk-prefetch into L2 the per-tile data of the tile a CTA one
// residency wave later will take, so its dependent loads hit L2.
// No tensor cores: this is a gather, not a dense contraction.  The extend is
// bound by its per-tile load chain overlapped with FP64 issue and shared-memory
// gathers, the laplace by load latency; DESIGN.md §Kernels has the measurements.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"

namespace cpm {
namespace {

// Degree-3 Lagrange weights on nodes (-1, 0, 1, 2) at t (reading R2),
// factored through q = t(t-1) and p = (t+1)(t-2)/2 = q/2 - 1:
//   w0 = -t(t-1)(t-2)/6 = q(2-t)/6    w1 = (t+1)(t-1)(t-2)/2 = p(t-1)
//   w2 = -(t+1)t(t-2)/2 = -p t        w3 = (t+1)t(t-1)/6 = q(t+1)/6
__device__ __forceinline__ void lagrange4(double t, double w[4]) {
  const double q = fma(t, t, -t);
  const double q6 = q * (1.0 / 6.0), q3 = q * (1.0 / 3.0);
  const double p = fma(q, 0.5, -1.0);
  w[0] = fma(-q6, t, q3);
  w[1] = fma(p, t, -p);
  w[2] = -p * t;
  w[3] = fma(q6, t, q6);
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ------------------------------------------------------------------ node-per-thread extend
// One CTA (128 threads) per tile, up to 4 eval nodes per thread, 8 CTAs per SM:
//   1. streaming loads of the tile's node offsets into registers (evict-first)
//   2. cp.async of the run descriptors into shared memory
//   3. cp.async of the box cells, 8 lanes per run (one coalesced 64-byte read)
//   4. per node: Lagrange weights from the offsets, x-y-z contraction -> vb
// The tile's nodes are sorted by stencil base, so the lanes of a half-warp read
// few distinct addresses (broadcast).  u is read with an evict-last L2 policy
// and vb written with one, so both stay resident in L2 for k_laplace.
constexpr int kNtThreads = 128;

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async8_hint(void* smem, const void* gmem, uint64_t pol) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "l"(pol));
}
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;\n"
               : "=d"(v)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_hint(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;\n"
               : "=r"(v)
               : "l"(p), "l"(pol));
  return v;
}
// L2 prefetch of the 16-byte granules inside [p, p + bytes) (rounded inward at the
// end, so it never reaches past the array; the start rounds down by < 16 bytes
// into the same allocation).
__device__ __forceinline__ void prefetch_l2_bytes(const void* p, size_t bytes) {
  const uintptr_t a0 = (uintptr_t)p & ~(uintptr_t)15;
  const uintptr_t a1 = ((uintptr_t)p + bytes) & ~(uintptr_t)15;
  if (a1 <= a0) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a0), "r"((unsigned)(a1 - a0))
               : "memory");
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// Slot s of a tile (thread tid handles slots tid + 128 k; build.cu k_warp_order):
// nodes 0 .. 2np-1 (equal-base pairs) one per slot, every adjacent lane pair reading
// one address (16 distinct doubles per warp: one wavefront); the nd unpaired nodes
// that complete the last pair warp two slots each (both lanes gather, the even one
// writes); the other unpaired nodes one per slot (32 distinct doubles, two
// wavefronts, but half the instructions of a duplicated node).
__device__ __forceinline__ int slot_node(int s, int np2, int nd, bool& write) {
  write = true;
  if (s < np2) return s;
  if (s < np2 + 2 * nd) {
    write = ((s - np2) & 1) == 0;
    return np2 + ((s - np2) >> 1);
  }
  return s - nd;
}

__device__ __forceinline__ void contract_node(const double (&tn)[3], uint32_t eo,
                                              const double* __restrict__ box, int sx, int sxy,
                                              double* __restrict__ out, bool write, uint64_t pol) {
  double wx[4], wy[4], wz[4];
  lagrange4(tn[0], wx);
  lagrange4(tn[1], wy);
  lagrange4(tn[2], wz);
  const double* p = box + (eo & 0xffffu);
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double accy = 0.0;
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) {
      const double* row = p + bb * sx + c * sxy;
      const double rx = (wx[0] * row[0] + wx[1] * row[1]) + (wx[2] * row[2] + wx[3] * row[3]);
      accy += wy[bb] * rx;
    }
    acc += wz[c] * accy;
  }
  if (write) st_hint(out + (eo >> 16), acc, pol);
}

template <bool ZERO, int MINB = 8, int kNtPre = 3, int FILL = 1>
__global__ void __launch_bounds__(kNtThreads, MINB)
    k_extend_nt(const TileHdr* __restrict__ tiles, int boxCells, int descCap,
                const uint64_t* __restrict__ runs, const double* __restrict__ u,
                const double* __restrict__ uh, uint32_t split, const double* __restrict__ tx,
                const double* __restrict__ ty, const double* __restrict__ tz,
                const uint32_t* __restrict__ eoff, double* __restrict__ vb,
                const int* __restrict__ skip, int pfd, int tbase, int tend) {
  // The band metadata (header, node offsets, run descriptors) is constant: it is
  // requested before pdl_wait(); u is read and vb written only after it.
  extern __shared__ double smn[];
  double* box = smn;
  uint64_t* desc = (uint64_t*)(box + boxCells);
  const int t = tbase + (int)blockIdx.x, tid = threadIdx.x;  // tiles [tbase, tend)
  const TileHdr* T = tiles + t;
  const int4 h0 = __ldg((const int4*)T), h1 = __ldg((const int4*)T + 1);  // e0 e1 a0 a1 | r0 r1 np pad2
  const int2 h2 = __ldg((const int2*)T->pad);                                // row, plane stride
  const int e0 = h0.x, ne = h0.y - e0, r0 = h1.x, r1 = h1.y;
  const int np2 = 2 * h1.z, nd = h1.w, nslot = ne + nd;
  const int sx = h2.x, sxy = h2.y;
  const uint64_t pfirst = policy_evict_first(), plast = policy_evict_last();
  // the first kNtPre slots of this thread are requested before the box is staged
  double nt[kNtPre][3];
  uint32_t eo[kNtPre];
#pragma unroll
  for (int k = 0; k < kNtPre; ++k) {
    const int sl = tid + k * kNtThreads;
    if (sl < nslot) {
      bool w;
      const int i = e0 + slot_node(sl, np2, nd, w);
      nt[k][0] = ld_hint(tx + i, pfirst);
      nt[k][1] = ld_hint(ty + i, pfirst);
      nt[k][2] = ld_hint(tz + i, pfirst);
      eo[k] = ld_hint(eoff + i, pfirst);
    }
  }
  if (ZERO) {
    const int nbox = sxy * T->sz;
    for (int c = tid; c < nbox; c += kNtThreads) box[c] = 0.0;
  }
  const int g = tid >> 3, l = tid & 7, g4 = tid >> 2, l4 = tid & 3;
  int nr = min(descCap, r1 - r0);
  for (int r = tid; r < nr; r += kNtThreads) cp_async8_hint(desc + r, runs + r0 + r, pfirst);
  cp_commit();
  pdl_wait();  // the predecessor grid (producer of u, reader of vb) has completed
  if (skip && *skip) {
    cp_wait<0>();
    return;
  }
  for (int c0 = r0; c0 < r1; c0 += nr, nr = min(descCap, r1 - c0)) {
    if (c0 > r0) {
      __syncthreads();  // previous round's descriptors consumed
      for (int r = tid; r < nr; r += kNtThreads) cp_async8_hint(desc + r, runs + c0 + r, pfirst);
      cp_commit();
    }
    cp_wait<0>();
    __syncthreads();  // descriptors landed (and the ZERO clear done)
    if (FILL == 1) {
      // 4 lanes per run, cells l and l + 4: 8 runs per warp iteration (the round-1 8 lanes
      // per run left half the lanes idle on runs of ~4 cells and doubled the loop's
      // issue: extend 117.1 -> 108.5 us at config 1)
      for (int r = g4; r < nr; r += kNtThreads / 4) {
        const uint64_t d = desc[r];
        const uint32_t src = (uint32_t)d, dst = (uint32_t)(d >> 32) & 0xffffu,
                       len = (uint32_t)(d >> 48) & 0xffu;
        const double* gsrc = src >= split ? uh + (src - split) : u + src;  // runs never straddle split
        if (l4 < len) cp_async8_hint(box + dst + l4, gsrc + l4, plast);
        if (l4 + 4 < len) cp_async8_hint(box + dst + l4 + 4, gsrc + l4 + 4, plast);
      }
    } else {
      for (int r = g; r < nr; r += kNtThreads / 8) {
        const uint64_t d = desc[r];
        const uint32_t src = (uint32_t)d, dst = (uint32_t)(d >> 32) & 0xffffu,
                       len = (uint32_t)(d >> 48) & 0xffu;
        if (l < len) {
          const double* gsrc = src >= split ? uh + (src - split) : u + src;  // runs never straddle split
          cp_async8_hint(box + dst + l, gsrc + l, plast);
        }
      }
    }
    cp_commit();
  }
  // The tile a CTA about one residency wave later will take (t + pfd): its
  // descriptors and node offsets into L2 now, so that CTA's dependent loads are
  // L2 hits (one lane; the header load it needs is itself that CTA's first load).
  if (tid == kNtThreads - 32 && t + pfd < tend) {
    const TileHdr* F = tiles + t + pfd;
    const int f0 = F->e0, f1 = F->e1, q0 = F->r0, q1 = F->r1;
    prefetch_l2_bytes(runs + q0, (size_t)(q1 - q0) * 8);
    prefetch_l2_bytes(tx + f0, (size_t)(f1 - f0) * 8);
    prefetch_l2_bytes(ty + f0, (size_t)(f1 - f0) * 8);
    prefetch_l2_bytes(tz + f0, (size_t)(f1 - f0) * 8);
    prefetch_l2_bytes(eoff + f0, (size_t)(f1 - f0) * 4);
    // and the header that lane will read one wave later
    if (t + 2 * pfd < tend) prefetch_l2_bytes(tiles + t + 2 * pfd, sizeof(TileHdr));
  }
  cp_wait<0>();
  __syncthreads();
  double* out = vb + (size_t)t * kBrickCells;
#pragma unroll
  for (int k = 0; k < kNtPre; ++k) {
    const int sl = tid + k * kNtThreads;
    if (sl < nslot) {
      bool w;
      slot_node(sl, np2, nd, w);
      contract_node(nt[k], eo[k], box, sx, sxy, out, w, plast);
    }
  }
  for (int sl = tid + kNtPre * kNtThreads; sl < nslot; sl += kNtThreads) {
    bool w;
    const int i = e0 + slot_node(sl, np2, nd, w);
    double tn[3] = {ld_hint(tx + i, pfirst), ld_hint(ty + i, pfirst), ld_hint(tz + i, pfirst)};
    contract_node(tn, ld_hint(eoff + i, pfirst), box, sx, sxy, out, w, plast);
  }
}

// ------------------------------------------------------------------ item extend
// The default extend (bands in item order, build.cu k_item_order): as k_extend_nt,
// but a lane evaluates an ITEM of one or two equal-base nodes, so each of its 64
// shared-memory gathers feeds two contractions; warp w takes the tile's rounds
// w, w + 4, ...  Per node the arithmetic is contract_node's, operation for
// operation, so E u is bit-identical to the pair order's.
struct ItemLane {
  int i;       // first node (absolute eval index), -1 = idle lane
  bool two;    // a second node at i + 1
};
__device__ __forceinline__ ItemLane item_of(uint64_t w, int e0, int lane) {
  ItemLane it;
  const uint32_t flags = (uint32_t)w;
  const int base = (int)((w >> 32) & 0xffffu), nv = (int)((w >> 48) & 0x3fu);
  it.i = lane < nv ? e0 + base + lane + __popc(flags & ((1u << lane) - 1u)) : -1;
  it.two = (flags >> lane) & 1u;
  return it;
}

__device__ __forceinline__ void contract_item(const double (&ta)[3], const double (&tb)[3], uint32_t eoa,
                                              uint32_t eob, bool two, const double* __restrict__ box, int sx,
                                              int sxy, double* __restrict__ out, uint64_t pol) {
  double ax[4], ay[4], az[4], bx[4], by[4], bz[4];
  lagrange4(ta[0], ax);
  lagrange4(ta[1], ay);
  lagrange4(ta[2], az);
  lagrange4(tb[0], bx);
  lagrange4(tb[1], by);
  lagrange4(tb[2], bz);
  const double* p = box + (eoa & 0xffffu);
  double acca = 0.0, accb = 0.0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double ya = 0.0, yb = 0.0;
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) {
      const double* row = p + bb * sx + c * sxy;
      const double r0 = row[0], r1 = row[1], r2 = row[2], r3 = row[3];
      ya += ay[bb] * ((ax[0] * r0 + ax[1] * r1) + (ax[2] * r2 + ax[3] * r3));
      yb += by[bb] * ((bx[0] * r0 + bx[1] * r1) + (bx[2] * r2 + bx[3] * r3));
    }
    acca += az[c] * ya;
    accb += bz[c] * yb;
  }
  st_hint(out + (eoa >> 16), acca, pol);
  if (two) st_hint(out + (eob >> 16), accb, pol);
}

template <bool ZERO, int MINB>
__global__ void __launch_bounds__(kNtThreads, MINB)
    k_extend_it(const TileHdr* __restrict__ tiles, int boxCells, int descCap,
                const uint64_t* __restrict__ runs, const double* __restrict__ u,
                const double* __restrict__ uh, uint32_t split, const double* __restrict__ tx,
                const double* __restrict__ ty, const double* __restrict__ tz,
                const uint32_t* __restrict__ eoff, const uint64_t* __restrict__ rnd,
                double* __restrict__ vb, const int* __restrict__ skip, int pfd, int tbase, int tend) {
  extern __shared__ double smn[];
  double* box = smn;
  uint64_t* desc = (uint64_t*)(box + boxCells);
  const int t = tbase + (int)blockIdx.x, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const TileHdr* T = tiles + t;
  const int e0 = T->e0, r0 = T->r0, r1 = T->r1;
  const int q0 = T->np, nq = T->pad2;
  const int sx = T->pad[0], sxy = T->pad[1];
  const uint64_t pfirst = policy_evict_first(), plast = policy_evict_last();
  // this warp's first round: its items' offsets are requested before the box is staged
  double ta[3] = {0.0, 0.0, 0.0}, tb[3] = {0.0, 0.0, 0.0};
  uint32_t eoa = 0, eob = 0;
  ItemLane it{-1, false};
  bool single = false;
  if (warp < nq) {
    const uint64_t w = __ldg(rnd + q0 + warp);
    single = (uint32_t)w == 0u;
    it = item_of(w, e0, lane);
    if (it.i >= 0) {
      const int j = it.two ? it.i + 1 : it.i;
      ta[0] = ld_hint(tx + it.i, pfirst);
      ta[1] = ld_hint(ty + it.i, pfirst);
      ta[2] = ld_hint(tz + it.i, pfirst);
      eoa = ld_hint(eoff + it.i, pfirst);
      tb[0] = ld_hint(tx + j, pfirst);
      tb[1] = ld_hint(ty + j, pfirst);
      tb[2] = ld_hint(tz + j, pfirst);
      eob = ld_hint(eoff + j, pfirst);
    }
  }
  if (ZERO) {
    const int nbox = sxy * T->sz;
    for (int c = tid; c < nbox; c += kNtThreads) box[c] = 0.0;
  }
  const int g = tid >> 3, l = tid & 7;
  int nr = min(descCap, r1 - r0);
  for (int r = tid; r < nr; r += kNtThreads) cp_async8_hint(desc + r, runs + r0 + r, pfirst);
  cp_commit();
  pdl_wait();
  if (skip && *skip) {
    cp_wait<0>();
    return;
  }
  for (int c0 = r0; c0 < r1; c0 += nr, nr = min(descCap, r1 - c0)) {
    if (c0 > r0) {
      __syncthreads();
      for (int r = tid; r < nr; r += kNtThreads) cp_async8_hint(desc + r, runs + c0 + r, pfirst);
      cp_commit();
    }
    cp_wait<0>();
    __syncthreads();
    for (int r = g; r < nr; r += kNtThreads / 8) {
      const uint64_t d = desc[r];
      const uint32_t src = (uint32_t)d, dst = (uint32_t)(d >> 32) & 0xffffu,
                     len = (uint32_t)(d >> 48) & 0xffu;
      if (l < len) {
        const double* gsrc = src >= split ? uh + (src - split) : u + src;
        cp_async8_hint(box + dst + l, gsrc + l, plast);
      }
    }
    cp_commit();
  }
  if (tid == kNtThreads - 32 && t + pfd < tend) {
    const TileHdr* F = tiles + t + pfd;
    const int f0 = F->e0, f1 = F->e1, fq0 = F->r0, fq1 = F->r1;
    prefetch_l2_bytes(runs + fq0, (size_t)(fq1 - fq0) * 8);
    prefetch_l2_bytes(tx + f0, (size_t)(f1 - f0) * 8);
    prefetch_l2_bytes(ty + f0, (size_t)(f1 - f0) * 8);
    prefetch_l2_bytes(tz + f0, (size_t)(f1 - f0) * 8);
    prefetch_l2_bytes(eoff + f0, (size_t)(f1 - f0) * 4);
    prefetch_l2_bytes(rnd + F->np, (size_t)F->pad2 * 8);
    if (t + 2 * pfd < tend) prefetch_l2_bytes(tiles + t + 2 * pfd, sizeof(TileHdr));
  }
  cp_wait<0>();
  __syncthreads();
  double* out = vb + (size_t)t * kBrickCells;
  // rounds without a two-node item (warp-uniform flags == 0) run the single contraction
  if (it.i >= 0) {
    if (single) contract_node(ta, eoa, box, sx, sxy, out, true, plast);
    else contract_item(ta, tb, eoa, eob, it.two, box, sx, sxy, out, plast);
  }
  for (int q = warp + kNtThreads / 32; q < nq; q += kNtThreads / 32) {
    const uint64_t w = __ldg(rnd + q0 + q);
    it = item_of(w, e0, lane);
    if (it.i >= 0) {
      const double a3[3] = {ld_hint(tx + it.i, pfirst), ld_hint(ty + it.i, pfirst), ld_hint(tz + it.i, pfirst)};
      const uint32_t ea = ld_hint(eoff + it.i, pfirst);
      if ((uint32_t)w == 0u) {
        contract_node(a3, ea, box, sx, sxy, out, true, plast);
      } else {
        const int j = it.two ? it.i + 1 : it.i;
        const double b3[3] = {ld_hint(tx + j, pfirst), ld_hint(ty + j, pfirst), ld_hint(tz + j, pfirst)};
        contract_item(a3, b3, ea, ld_hint(eoff + j, pfirst), it.two, box, sx, sxy, out, plast);
      }
    }
  }
}

// Dense halo brick: cell (x, y, z), x, y, z in -1..8, at (x+1) + 10 (y+1) + 100 (z+1).
__device__ __forceinline__ int hidx(int x, int y, int z) { return (x + 1) + 10 * (y + 1) + 100 * (z + 1); }


// One CTA per tile.  vb holds E u per brick cell (t * 512 + cell, written by
// k_extend_nt), so every global load of a CTA is one step from its header:
// the own eval cells, the neighbours' face layers under own eval cells, and the
// output nodes' u and cells; then one barrier and the 7-point combination.
template <int kLapThreads>
__global__ void __launch_bounds__(kLapThreads) k_laplace(const TileHdr* __restrict__ tiles,
                                                         const double* __restrict__ u,
                                                         const uint16_t* __restrict__ acell,
                                                         const double* __restrict__ vb,
                                                         double* __restrict__ y, double diag,
                                                         double ih2,
                                                         const double* __restrict__ scale, int lds,
                                                         const int* __restrict__ skip, int pfd) {
  __shared__ double E[1000];
  // tiles in reverse order: the extend's last tiles (their E u, u) are the ones
  // still in L2 when this kernel starts
  const int t = (int)gridDim.x - 1 - (int)blockIdx.x, tid = threadIdx.x;
  const TileHdr* T = tiles + t;
  const int a0 = T->a0, a1 = T->a1;
  if (a0 == a1) return;
  if (tid == kLapThreads - 32 && t - pfd >= 0) {  // a later CTA's tile into L2
    const TileHdr* F = tiles + t - pfd;
    const int f0 = F->a0, f1 = F->a1;
    prefetch_l2_bytes(acell + f0, (size_t)(f1 - f0) * 2);
    prefetch_l2_bytes(u + f0, (size_t)(f1 - f0) * 8);
    prefetch_l2_bytes(vb + (size_t)(t - pfd) * kBrickCells, kBrickCells * 8);
  }
  constexpr int kOut = kBrickCells / kLapThreads;
  // output nodes: up to kOut per thread; their cells (band metadata) are read
  // before pdl_wait(), u and E u after it
  int ac[kOut];
  double au[kOut];
#pragma unroll
  for (int k = 0; k < kOut; ++k) {
    const int a = a0 + tid + k * kLapThreads;
    if (a < a1) ac[k] = __ldg(acell + a);
  }
  pdl_wait();  // the extend (E u) and the producer of u have completed
  if (skip && *skip) return;
#pragma unroll
  for (int k = 0; k < kOut; ++k) {
    const int a = a0 + tid + k * kLapThreads;
    if (a < a1) au[k] = __ldg(u + a);
  }
  // own eval cells (the only cells the extend wrote)
  const double* vt = vb + (size_t)t * kBrickCells;
#pragma unroll
  for (int k = 0; k < kBrickCells / kLapThreads; ++k) {
    const int c = tid + k * kLapThreads;
    if ((T->emask[c >> 5] >> (c & 31)) & 1u) E[hidx(c & 7, (c >> 3) & 7, c >> 6)] = __ldg(vt + c);
  }
  // 6 x 64 face cells of the neighbours, read where the own boundary cell is an eval cell
  // (every 6-neighbour of an active node is an eval node, Sigma_G of reading R1)
#pragma unroll
  for (int k = 0; k < (384 + kLapThreads - 1) / kLapThreads; ++k) {
    const int q = tid + k * kLapThreads;
    if (q < 384) {
      const int f = q >> 6, i = q & 7, j = (q >> 3) & 7;
      const int src = T->nbr[f];
      if (src >= 0) {
        const int axis = f >> 1, plus = (f & 1) == 0;
        const int in = plus ? 0 : 7;    // layer read in the neighbour
        const int me = plus ? 7 : 0;    // own boundary layer
        const int out = plus ? 8 : -1;  // halo layer written here
        int c, co, h;
        if (axis == 0) { c = in + 8 * i + 64 * j; co = me + 8 * i + 64 * j; h = hidx(out, i, j); }
        else if (axis == 1) { c = i + 8 * in + 64 * j; co = i + 8 * me + 64 * j; h = hidx(i, out, j); }
        else { c = i + 8 * j + 64 * in; co = i + 8 * j + 64 * me; h = hidx(i, j, out); }
        if ((T->emask[co >> 5] >> (co & 31)) & 1u) E[h] = __ldg(vb + (size_t)src * kBrickCells + c);
      }
    }
  }
  __syncthreads();
  const double s = scale ? __ldg(scale + (size_t)T->pad[2] * lds) : 1.0;
#pragma unroll
  for (int k = 0; k < kOut; ++k) {
    const int a = a0 + tid + k * kLapThreads;
    if (a < a1) {
      const int c = ac[k];
      const int h = hidx(c & 7, (c >> 3) & 7, c >> 6);
      const double sum = E[h + 1] + E[h - 1] + E[h + 10] + E[h - 10] + E[h + 100] + E[h - 100];
      y[a] = s * (diag * au[k] - ih2 * sum);
    }
  }
}


// ------------------------------------------------------------------ TMA laplace
// One CTA (128 threads) per tile; every E u load is a TMA copy issued by one
// thread after pdl_wait(): the own brick (4 KB bulk copy of vb slot t), the two
// z face layers of the z neighbours (512 B bulk copies), the y face layers (tensor
// copy, box 8 x 1 x 8 of the neighbour's brick) and the x face layers (tensor copy,
// box 2 x 8 x 8: 16-byte inner extent, the wanted layer and one more).  The copies
// land on one mbarrier; no per-element global loads, no emask test.  Then the
// 7-point combination in the same operation order as k_laplace (bit-identical).
__device__ __forceinline__ unsigned sm32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tma_bulk(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sm32(dst)),
      "l"(src), "r"(bytes), "r"(sm32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_4d(void* dst, const CUtensorMap* tm, int x, int y, int z, int t, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(sm32(dst)),
      "l"(tm), "r"(x), "r"(y), "r"(z), "r"(t), "r"(sm32(bar))
      : "memory");
}

__global__ void __launch_bounds__(128, 16) k_laplace_tma(const TileHdr* __restrict__ tiles, const double* __restrict__ u,
                                                     const uint16_t* __restrict__ acell,
                                                     const double* __restrict__ vb, double* __restrict__ y,
                                                     double diag, double ih2, const double* __restrict__ scale,
                                                     int lds, const int* __restrict__ skip, int pfd,
                                                     const __grid_constant__ CUtensorMap tmX,
                                                     const __grid_constant__ CUtensorMap tmY) {
  __shared__ __align__(128) double own[512];
  __shared__ __align__(128) double fx[2][128];  // [+x, -x] box 2 x 8 x 8: x + 2 y + 16 z
  __shared__ __align__(128) double fy[2][64];   // [+y, -y] box 8 x 1 x 8: x + 8 z
  __shared__ __align__(128) double fz[2][64];   // [+z, -z] layer: x + 8 y
  __shared__ uint64_t bar;
  const int t = (int)gridDim.x - 1 - (int)blockIdx.x, tid = threadIdx.x;
  const TileHdr* T = tiles + t;
  const int4 h0 = __ldg((const int4*)T);  // e0 e1 a0 a1
  const int a0 = h0.z, a1 = h0.w;
  if (a0 == a1) return;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sm32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid == 32 && t - pfd >= 0) {  // a later CTA's tile into L2
    const TileHdr* F = tiles + t - pfd;
    const int f0 = F->a0, f1 = F->a1;
    prefetch_l2_bytes(acell + f0, (size_t)(f1 - f0) * 2);
    prefetch_l2_bytes(u + f0, (size_t)(f1 - f0) * 8);
    prefetch_l2_bytes(vb + (size_t)(t - pfd) * kBrickCells, kBrickCells * 8);
  }
  int ac[4];
  double au[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int a = a0 + tid + k * 128;
    if (a < a1) ac[k] = __ldg(acell + a);
  }
  __syncthreads();  // mbarrier initialised
  pdl_wait();       // the extend (E u) and the producer of u have completed
  if (skip && *skip) return;
  if (tid == 0) {
    int nb[6];
    unsigned bytes = kBrickCells * 8;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      nb[f] = T->nbr[f];
      if (nb[f] >= 0) bytes += f < 2 ? 1024u : 512u;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm32(&bar)), "r"(bytes)
                 : "memory");
    tma_bulk(own, vb + (size_t)t * kBrickCells, kBrickCells * 8, &bar);
    if (nb[0] >= 0) tma_4d(fx[0], &tmX, 0, 0, 0, nb[0], &bar);  // +x neighbour: its x = 0 layer
    if (nb[1] >= 0) tma_4d(fx[1], &tmX, 6, 0, 0, nb[1], &bar);  // -x neighbour: x = 7 (box x = 6, 7)
    if (nb[2] >= 0) tma_4d(fy[0], &tmY, 0, 0, 0, nb[2], &bar);
    if (nb[3] >= 0) tma_4d(fy[1], &tmY, 0, 7, 0, nb[3], &bar);
    if (nb[4] >= 0) tma_bulk(fz[0], vb + (size_t)nb[4] * kBrickCells, 512, &bar);
    if (nb[5] >= 0) tma_bulk(fz[1], vb + (size_t)nb[5] * kBrickCells + 448, 512, &bar);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int a = a0 + tid + k * 128;
    if (a < a1) au[k] = __ldg(u + a);
  }
  const double s = scale ? __ldg(scale + (size_t)T->pad[2] * lds) : 1.0;
  asm volatile(
      "{\n .reg .pred p;\n WAITL_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      " @!p bra WAITL_%=;\n}\n" ::"r"(sm32(&bar))
      : "memory");
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int a = a0 + tid + k * 128;
    if (a < a1) {
      const int c = ac[k], x = c & 7, yy = (c >> 3) & 7, z = c >> 6;
      const double xp = x < 7 ? own[c + 1] : fx[0][2 * yy + 16 * z];
      const double xm = x > 0 ? own[c - 1] : fx[1][1 + 2 * yy + 16 * z];
      const double yp = yy < 7 ? own[c + 8] : fy[0][x + 8 * z];
      const double ym = yy > 0 ? own[c - 8] : fy[1][x + 8 * z];
      const double zp = z < 7 ? own[c + 64] : fz[0][x + 8 * yy];
      const double zm = z > 0 ? own[c - 64] : fz[1][x + 8 * yy];
      const double sum = xp + xm + yp + ym + zp + zm;
      y[a] = s * (diag * au[k] - ih2 * sum);
    }
  }
}

// ------------------------------------------------------------------ fused apply (experiment)
// One CTA (128 threads) per tile, no vb: stage the FUSED box (build.cu build_fused:
// the stencils of the tile's eval nodes and of its halo nodes, the face-neighbour
// eval nodes next to its active nodes), contract the own eval nodes (pair order of
// k_extend_nt) and the halo nodes into the dense 10^3 halo brick in shared memory,
// then the 7-point combination for the tile's output nodes.  E u never leaves the SM;
// the price is the halo nodes' second evaluation.
__device__ __forceinline__ double contract_val(double tnx, double tny, double tnz, const double* __restrict__ p,
                                               int sx, int sxy) {
  double wx[4], wy[4], wz[4];
  lagrange4(tnx, wx);
  lagrange4(tny, wy);
  lagrange4(tnz, wz);
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double accy = 0.0;
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) {
      const double* row = p + bb * sx + c * sxy;
      const double rx = (wx[0] * row[0] + wx[1] * row[1]) + (wx[2] * row[2] + wx[3] * row[3]);
      accy += wy[bb] * rx;
    }
    acc += wz[c] * accy;
  }
  return acc;
}

__global__ void __launch_bounds__(kNtThreads, 6)
    k_apply_fused(const TileHdr* __restrict__ ftiles, int boxCells, int descCap, const uint64_t* __restrict__ runs,
                  const double* __restrict__ u, const double* __restrict__ tx, const double* __restrict__ ty,
                  const double* __restrict__ tz, const uint32_t* __restrict__ feoff, const int* __restrict__ hst,
                  const uint64_t* __restrict__ halo, const uint16_t* __restrict__ acell, double* __restrict__ y,
                  double diag, double ih2, const double* __restrict__ scale, int lds, const int* __restrict__ skip) {
  extern __shared__ double smf[];
  double* box = smf;
  uint64_t* desc = (uint64_t*)(box + boxCells);
  __shared__ double E[1000];
  const int t = blockIdx.x, tid = threadIdx.x;
  const TileHdr* T = ftiles + t;
  const int e0 = T->e0, ne = T->e1 - e0, r0 = T->r0, r1 = T->r1;
  const int np2 = 2 * T->np, nd = T->pad2, nslot = ne + nd;
  const int sx = T->pad[0], sxy = T->pad[1];
  const int h0 = hst[t], nh = hst[t + 1] - h0;
  const int a0 = T->a0, a1 = T->a1;
  const int g = tid >> 3, l = tid & 7;
  int nr = min(descCap, r1 - r0);
  for (int r = tid; r < nr; r += kNtThreads) cp_async8_hint(desc + r, runs + r0 + r, policy_evict_first());
  cp_commit();
  pdl_wait();
  if (skip && *skip) {
    cp_wait<0>();
    return;
  }
  const uint64_t plast = policy_evict_last();
  for (int c0 = r0; c0 < r1; c0 += nr, nr = min(descCap, r1 - c0)) {
    if (c0 > r0) {
      __syncthreads();
      for (int r = tid; r < nr; r += kNtThreads) cp_async8_hint(desc + r, runs + c0 + r, policy_evict_first());
      cp_commit();
    }
    cp_wait<0>();
    __syncthreads();
    for (int r = g; r < nr; r += kNtThreads / 8) {
      const uint64_t d = desc[r];
      const uint32_t src = (uint32_t)d, dst = (uint32_t)(d >> 32) & 0xffffu, len = (uint32_t)(d >> 48) & 0xffu;
      if (l < len) cp_async8_hint(box + dst + l, u + src + l, plast);
    }
    cp_commit();
  }
  cp_wait<0>();
  __syncthreads();
  // own eval nodes (k_extend_nt's slot order) -> E at their brick cells
  for (int sl = tid; sl < nslot; sl += kNtThreads) {
    bool w;
    const int i = e0 + slot_node(sl, np2, nd, w);
    const uint32_t eo = __ldg(feoff + i);
    const double v = contract_val(__ldg(tx + i), __ldg(ty + i), __ldg(tz + i), box + (eo & 0xffffu), sx, sxy);
    const int c = (int)(eo >> 16);
    if (w) E[hidx(c & 7, (c >> 3) & 7, c >> 6)] = v;
  }
  // halo nodes (the neighbours' eval nodes next to own active nodes) -> E halo layer
  for (int k = tid; k < nh; k += kNtThreads) {
    const uint64_t hv = __ldg(halo + h0 + k);
    const int i = (int)(uint32_t)hv;
    const uint32_t off = (uint32_t)(hv >> 32) & 0xffffu;
    E[(int)(hv >> 48)] = contract_val(__ldg(tx + i), __ldg(ty + i), __ldg(tz + i), box + off, sx, sxy);
  }
  __syncthreads();
  const double s = scale ? __ldg(scale + (size_t)T->pad[2] * lds) : 1.0;
  for (int a = a0 + tid; a < a1; a += kNtThreads) {
    const int c = __ldg(acell + a);
    const int h = hidx(c & 7, (c >> 3) & 7, c >> 6);
    const double sum = E[h + 1] + E[h - 1] + E[h + 10] + E[h - 10] + E[h + 100] + E[h - 100];
    y[a] = s * (diag * __ldg(u + a) - ih2 * sum);
  }
}

}  // namespace

int apply_device(const cpm_band* b, double c, const double* u, double* y, const double* scale,
                 int lds, cudaStream_t s, const int* skip) {
  return apply_device_split(b, c, u, u, y, scale, lds, s, skip);
}

// The extend's E u writes and the laplace's reads of vb run under an L2
// access-policy window (persisting lines in the set-aside L2 of
// cudaLimitPersistingL2CacheSize), so the E u round trip mostly stays in L2:
// in-situ DRAM traffic per config-1 apply 404 -> 313 MB, time unchanged (neither
// kernel is DRAM-bound).  CPM_L2_PERSIST=0 disables it (A/B).
L2Window vb_window(const cpm_band* b) {
  static const size_t cap = []() -> size_t {
    const char* v = getenv("CPM_L2_PERSIST");
    if (v && *v == '0') return 0;
    int dev = 0, maxp = 0, maxw = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (maxp <= 0 || maxw <= 0) return 0;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return std::min((size_t)maxp, (size_t)maxw);
  }();
  L2Window w;
  if (!cap || !b->vb) return w;
  const size_t bytes = sizeof(double) * kBrickCells * (size_t)b->nT;
  w.base = b->vb;
  w.bytes = std::min(bytes, cap);
  w.hit = (float)std::min(1.0, (double)cap / (double)w.bytes);
  return w;
}

namespace {
// L2 prefetch distance in tiles (both kernels): one wave of resident extend CTAs,
// 8 per SM (measured: 0.5x and 2x are slower; CPM_EXT_PFD / CPM_LAP_PFD override)
int prefetch_distance() {
  static const int pfd = [] {
    const char* v = getenv("CPM_EXT_PFD");
    if (v) return atoi(v);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return 8 * sms;
  }();
  return pfd;
}
}  // namespace

int extend_tiles(const cpm_band* b, const double* u, const double* uh, cudaStream_t s, const int* skip,
                 int t0, int t1) {
  if (t1 <= t0) return CPM_OK;
  const int pfd = prefetch_distance();
  // descriptors staged per round: 256 (2 KB) lets 9 CTAs per SM fit next to the largest config-1 box
  static const int descCap = getenv("CPM_DESC_CAP") ? atoi(getenv("CPM_DESC_CAP")) : 256;
  // CPM_EXT_SMEM_PAD (bytes, experiment): extra dynamic shared memory per CTA, to
  // measure the extend's sensitivity to resident CTAs per SM
  static const size_t smpad = getenv("CPM_EXT_SMEM_PAD") ? (size_t)atol(getenv("CPM_EXT_SMEM_PAD")) : 0;
  const size_t smem = (size_t)b->maxBox * 8 + (size_t)descCap * 8 + smpad;
  ProfScope ps(K_EXTEND, s);
#define CPM_EXTNT(Z, MB, PRE, F4)                                                              \
  do {                                                                                       \
    static bool attr = false;                                                                \
    if (!attr) {                                                                             \
      CPM_CUDA(cudaFuncSetAttribute(k_extend_nt<Z, MB, PRE, F4>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                    227 * 1024));                                            \
      attr = true;                                                                           \
    }                                                                                        \
    CPM_CUDA(launch_pdl_l2(vb_window(b), k_extend_nt<Z, MB, PRE, F4>, dim3((unsigned)(t1 - t0)), dim3(kNtThreads), smem, s, \
                        b->tiles, (int)b->maxBox, descCap, (const uint64_t*)b->runs, u, uh,     \
                        (uint32_t)b->srcSplit, (const double*)b->tx, (const double*)b->ty,      \
                        (const double*)b->tz, (const uint32_t*)b->eoff, b->vb, skip, pfd, t0, t1)); \
  } while (0)
#define CPM_EXTIT(Z, MB)                                                                       \
  do {                                                                                       \
    static bool attr = false;                                                                \
    if (!attr) {                                                                             \
      CPM_CUDA(cudaFuncSetAttribute(k_extend_it<Z, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                    227 * 1024));                                            \
      attr = true;                                                                           \
    }                                                                                        \
    CPM_CUDA(launch_pdl_l2(vb_window(b), k_extend_it<Z, MB>, dim3((unsigned)(t1 - t0)), dim3(kNtThreads), smem, s, \
                        b->tiles, (int)b->maxBox, descCap, (const uint64_t*)b->runs, u, uh,     \
                        (uint32_t)b->srcSplit, (const double*)b->tx, (const double*)b->ty,      \
                        (const double*)b->tz, (const uint32_t*)b->eoff, (const uint64_t*)b->rnd, \
                        b->vb, skip, pfd, t0, t1));                                              \
  } while (0)
  static const int minb = getenv("CPM_IT_MINB") ? atoi(getenv("CPM_IT_MINB")) : 6;
  if (b->itemOrder) {
    if (minb == 8) {
      if (b->zeroFill) CPM_EXTIT(true, 8); else CPM_EXTIT(false, 8);
    } else if (minb == 7) {
      if (b->zeroFill) CPM_EXTIT(true, 7); else CPM_EXTIT(false, 7);
    } else {
      if (b->zeroFill) CPM_EXTIT(true, 6); else CPM_EXTIT(false, 6);
    }
  } else {
    // default: 56 registers (9 CTAs per SM), 2 slots' offsets prefetched (config 1:
    // 119.4 -> 117.1 us against 64 registers / 8 CTAs / 3 slots); CPM_NT_CFG=0: the
    // latter, 2: 9 CTAs with 3 slots (118.9 us)
    static const int cfg = getenv("CPM_NT_CFG") ? atoi(getenv("CPM_NT_CFG")) : 1;
    static const int fill = getenv("CPM_FILL") ? atoi(getenv("CPM_FILL")) : 1;  // 0: 8 lanes per run
    if (cfg == 0) {
      if (b->zeroFill) CPM_EXTNT(true, 8, 3, 0); else CPM_EXTNT(false, 8, 3, 0);
    } else if (cfg == 2) {
      if (b->zeroFill) CPM_EXTNT(true, 9, 3, 0); else CPM_EXTNT(false, 9, 3, 0);
    } else if (fill == 1) {
      if (b->zeroFill) CPM_EXTNT(true, 9, 2, 1); else CPM_EXTNT(false, 9, 2, 1);
    } else {
      if (b->zeroFill) CPM_EXTNT(true, 9, 2, 0); else CPM_EXTNT(false, 9, 2, 0);
    }
  }
#undef CPM_EXTNT
#undef CPM_EXTIT
  count_launch();
  CPM_CUDA(cudaGetLastError());
  return CPM_OK;
}

// Tensor maps over vb viewed as [nT][8][8][8] doubles (x fastest) for the TMA
// laplace's face copies: box 2 x 8 x 8 (x faces) and 8 x 1 x 8 (y faces).  Built
// once per band (vb and nT are fixed), cached in the band.
static int laplace_tmaps(const cpm_band* b) {
  if (b->tmReady) return CPM_OK;
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn enc = []() -> EncodeFn {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return (EncodeFn)fn;
  }();
  if (!enc) return fail(CPM_ERR_CUDA, "laplace: cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[4] = {8, 8, 8, (cuuint64_t)b->nT};
  const cuuint64_t strides[3] = {64, 512, 4096};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const cuuint32_t boxX[4] = {2, 8, 8, 1}, boxY[4] = {8, 1, 8, 1};
  CUtensorMap mx, my;
  for (int q = 0; q < 2; ++q) {
    const CUresult r = enc(q ? &my : &mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, b->vb, dims, strides,
                           q ? boxY : boxX, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(CPM_ERR_CUDA, "laplace: tensor map encoding failed");
  }
  cpm_band* mb = const_cast<cpm_band*>(b);
  std::memcpy(mb->tmX, &mx, sizeof(CUtensorMap));
  std::memcpy(mb->tmY, &my, sizeof(CUtensorMap));
  mb->tmReady = true;
  return CPM_OK;
}

int laplace_tiles(const cpm_band* b, double c, const double* u, double* y, const double* scale, int lds,
                  cudaStream_t s, const int* skip) {
  if (b->nT == 0) return CPM_OK;  // no tiles: no outputs (and no tensor map over an empty vb)
  const double ih2 = 1.0 / (b->h * b->h);
  const double diag = c + 6.0 * ih2;
  ProfScope ps(K_LAPLACE, s);
  // 128 threads per tile: 16 resident tiles per SM keep enough loads in flight
  static const int pfd2 = getenv("CPM_LAP_PFD") ? atoi(getenv("CPM_LAP_PFD")) : prefetch_distance();
  static const bool tma = !(getenv("CPM_LAP_TMA") && *getenv("CPM_LAP_TMA") == '0');
  if (tma) {
    CPM_TRY(laplace_tmaps(b));
    CUtensorMap mx, my;
    std::memcpy(&mx, b->tmX, sizeof(CUtensorMap));
    std::memcpy(&my, b->tmY, sizeof(CUtensorMap));
    // one tile per CTA (two tiles per CTA, both tiles' copies in flight before the
    // first wait: 45.5 us against 35.5, measured)
    CPM_CUDA(launch_pdl_l2(vb_window(b), k_laplace_tma, dim3((unsigned)b->nT), dim3(128), 0, s, b->tiles, u,
                           (const uint16_t*)b->acell, (const double*)b->vb, y, diag, ih2, scale, lds, skip, pfd2,
                           mx, my));
    count_launch();
    CPM_CUDA(cudaGetLastError());
    return CPM_OK;
  }
  CPM_CUDA(launch_pdl_l2(vb_window(b), k_laplace<128>, dim3((unsigned)b->nT), dim3(128), 0, s, b->tiles, u,
                      (const uint16_t*)b->acell, (const double*)b->vb, y, diag, ih2, scale, lds,
                      skip, pfd2));
  count_launch();
  CPM_CUDA(cudaGetLastError());
  return CPM_OK;
}

int apply_device_split(const cpm_band* b, double c, const double* u, const double* uh, double* y,
                       const double* scale, int lds, cudaStream_t s, const int* skip) {
  if (b->nT == 0) return CPM_OK;  // no tiles (an empty sub-band): nothing to write
  if (b->fzT) {  // the fused single-kernel apply (bands built with CPM_FUSED=1)
    const double ih2 = 1.0 / (b->h * b->h);
    const int descCap = 512;
    const size_t smem = (size_t)b->fzMaxBox * 8 + (size_t)descCap * 8;
    static bool attr = false;
    if (!attr) {
      CPM_CUDA(cudaFuncSetAttribute(k_apply_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
    ProfScope ps(K_EXTEND, s);
    CPM_CUDA(launch_pdl(k_apply_fused, dim3((unsigned)b->nT), dim3(kNtThreads), smem, s, (const TileHdr*)b->fzT,
                        b->fzMaxBox, descCap, (const uint64_t*)b->fzRuns, u, (const double*)b->tx,
                        (const double*)b->ty, (const double*)b->tz, (const uint32_t*)b->fzEoff,
                        (const int*)b->fzH, (const uint64_t*)b->fzHalo, (const uint16_t*)b->acell, y,
                        c + 6.0 * ih2, ih2, scale, lds, skip));
    count_launch();
    CPM_CUDA(cudaGetLastError());
    return CPM_OK;
  }
  CPM_TRY(extend_tiles(b, u, uh, s, skip, 0, b->nT));
  return laplace_tiles(b, c, u, y, scale, lds, s, skip);
}

}  // namespace cpm
