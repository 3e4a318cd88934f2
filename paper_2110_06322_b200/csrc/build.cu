// build.cu — band construction on the GPU (north_star item 1).
//
// Pipeline (all on the caller's stream):
//   B1  brick candidates: every 8^3 brick of the surface's padded box whose
//       centre lies within lambda + h + half-diagonal of the surface (the
//       distance function is 1-Lipschitz, so no band or ghost node is missed)
//   B2  radix-sort candidate bricks by Morton code (band order, reading R8)
//   B3  classify the 512 nodes of each candidate: Sigma_A (dist <= lambda,
//       inside [-L, L]^3) and Sigma_G (not in Sigma_A, a 6-neighbour in it);
//       per-brick 512-bit masks and counts
//   B4  scans -> tile slots, active/eval/ghost starts
//   B5  per node: closest point, stencil base floor(cp/h) - 1, offset
//       t = cp/h - floor(cp/h) (reading R2); coordinates for the caller
//   B6  dense brick map (bucketed node -> lattice index map), per-tile stencil
//       box and face neighbours, per-node box offsets, stencil coverage check
//   B7  stencil-box fill runs (consecutive band-order sources -> box rows)
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <memory>
#include <cstdio>
#include <cstring>
#include <vector>

#include "geom.cuh"
#include "internal.cuh"

namespace cpm {
namespace {

struct BuildParams {
  Surface s;
  double h, lam, slack;
  int M;
  int blo[3], bdim[3];  // brick box
};

// ------------------------------------------------------------------ B1
__global__ void k_brick_candidates(BuildParams P, uint64_t* keys, int* count) {
  int64_t n = (int64_t)P.bdim[0] * P.bdim[1] * P.bdim[2];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int bx = (int)(t % P.bdim[0]) + P.blo[0];
    int by = (int)((t / P.bdim[0]) % P.bdim[1]) + P.blo[1];
    int bz = (int)(t / ((int64_t)P.bdim[0] * P.bdim[1])) + P.blo[2];
    double cx = (bx * 8 + 3.5) * P.h, cy = (by * 8 + 3.5) * P.h, cz = (bz * 8 + 3.5) * P.h;
    double d = surface_dist(P.s, cx, cy, cz);
    // conservative: half-diagonal 3.5*sqrt(3)*h, plus one h for ghosts
    if (!(d <= P.lam + P.h + 3.5 * 1.7320508075688772 * P.h + P.slack)) continue;
    int slot = atomicAdd(count, 1);
    keys[slot] = brick_morton(bx, by, bz);
  }
}

__device__ inline bool in_domain(int i, int j, int k, int M) {
  return i >= -M && i <= M && j >= -M && j <= M && k >= -M && k <= M;
}

__device__ inline bool is_active(const BuildParams& P, int i, int j, int k) {
  if (!in_domain(i, j, k, P.M)) return false;
  double d = surface_dist(P.s, lat(i, P.h), lat(j, P.h), lat(k, P.h));
  return d <= P.lam;
}

// ------------------------------------------------------------------ B3
// One CTA of 512 threads per candidate brick; thread = cell lx + 8 ly + 64 lz.
__global__ void __launch_bounds__(512) k_classify(BuildParams P, const uint64_t* keys,
                                                  uint32_t* amask, uint32_t* gmask, int* na,
                                                  int* ng, int* ne) {
  int b = blockIdx.x;
  int bx, by, bz;
  morton_brick(keys[b], &bx, &by, &bz);
  int c = threadIdx.x;
  int i = bx * 8 + (c & 7), j = by * 8 + ((c >> 3) & 7), k = bz * 8 + (c >> 6);
  bool a = is_active(P, i, j, k);
  bool g = false;
  if (!a) {
    g = is_active(P, i + 1, j, k) || is_active(P, i - 1, j, k) || is_active(P, i, j + 1, k) ||
        is_active(P, i, j - 1, k) || is_active(P, i, j, k + 1) || is_active(P, i, j, k - 1);
  }
  uint32_t am = __ballot_sync(0xffffffffu, a);
  uint32_t gm = __ballot_sync(0xffffffffu, g);
  __shared__ int sa[16], sg[16];
  int w = c >> 5;
  if ((c & 31) == 0) {
    amask[(size_t)b * 16 + w] = am;
    gmask[(size_t)b * 16 + w] = gm;
    sa[w] = __popc(am);
    sg[w] = __popc(gm);
  }
  __syncthreads();
  if (c == 0) {
    int ta = 0, tg = 0;
    for (int q = 0; q < 16; ++q) {
      ta += sa[q];
      tg += sg[q];
    }
    na[b] = ta;
    ng[b] = tg;
    ne[b] = ta + tg;
  }
}

__device__ inline int mask_rank(const uint32_t* m16, int cell) {
  int w = cell >> 5, r = 0;
  for (int q = 0; q < w; ++q) r += __popc(m16[q]);
  return r + __popc(m16[w] & ((1u << (cell & 31)) - 1u));
}
__device__ inline bool mask_has(const uint32_t* m16, int cell) {
  return (m16[cell >> 5] >> (cell & 31)) & 1u;
}

// ------------------------------------------------------------------ B4 helpers
__global__ void k_compact_tiles(int nb, const int* ne, const int* tslot, const int* na,
                                const int* ng, const int* astart, const int* gstart,
                                const int* estart, const uint64_t* keys, const uint32_t* amask,
                                const uint32_t* gmask, TileHdr* tiles, uint32_t* tam,
                                uint32_t* tgm, int* tgstart) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb || ne[b] == 0) return;
  int t = tslot[b];
  TileHdr T;
  memset(&T, 0, sizeof(T));
  T.e0 = estart[b];
  T.e1 = estart[b] + ne[b];
  T.a0 = astart[b];
  T.a1 = astart[b] + na[b];
  morton_brick(keys[b], &T.bx, &T.by, &T.bz);
  for (int q = 0; q < 6; ++q) T.nbr[q] = -1;
  tgstart[t] = gstart[b];
  for (int q = 0; q < 16; ++q) {
    tam[(size_t)t * 16 + q] = amask[(size_t)b * 16 + q];
    tgm[(size_t)t * 16 + q] = gmask[(size_t)b * 16 + q];
    T.emask[q] = amask[(size_t)b * 16 + q] | gmask[(size_t)b * 16 + q];
  }
  tiles[t] = T;
}

// ------------------------------------------------------------------ B5
// One CTA (512 threads) per tile.  Eval order inside a tile: Sigma_A cells in
// lexicographic order, then Sigma_G cells.
__global__ void __launch_bounds__(512) k_node_data(BuildParams P, const TileHdr* tiles,
                                                   const uint32_t* tam, const uint32_t* tgm,
                                                   const int* tgstart, int32_t* aijk,
                                                   int32_t* gijk, uint16_t* acell, double* tx,
                                                   double* ty, double* tz, int32_t* ebase,
                                                   uint16_t* ecell, int* err) {
  int t = blockIdx.x;
  __shared__ uint32_t am[16], gm[16];
  if (threadIdx.x < 16) {
    am[threadIdx.x] = tam[(size_t)t * 16 + threadIdx.x];
    gm[threadIdx.x] = tgm[(size_t)t * 16 + threadIdx.x];
  }
  __syncthreads();
  const TileHdr T = tiles[t];
  int c = threadIdx.x;
  bool a = mask_has(am, c), g = mask_has(gm, c);
  if (!a && !g) return;
  int i = T.bx * 8 + (c & 7), j = T.by * 8 + ((c >> 3) & 7), k = T.bz * 8 + (c >> 6);
  int e;
  if (a) {
    int ra = mask_rank(am, c);
    int ai = T.a0 + ra;
    aijk[3 * (size_t)ai + 0] = i;
    aijk[3 * (size_t)ai + 1] = j;
    aijk[3 * (size_t)ai + 2] = k;
    acell[ai] = (uint16_t)c;
    e = T.e0 + ra;
  } else {
    int rg = mask_rank(gm, c);
    int gi = tgstart[t] + rg;
    gijk[3 * (size_t)gi + 0] = i;
    gijk[3 * (size_t)gi + 1] = j;
    gijk[3 * (size_t)gi + 2] = k;
    e = T.e0 + (T.a1 - T.a0) + rg;
  }
  double cx, cy, cz, d;
  bool ok = closest_point(P.s, lat(i, P.h), lat(j, P.h), lat(k, P.h), &cx, &cy, &cz, &d);
  if (!ok || !isfinite(cx) || !isfinite(cy) || !isfinite(cz)) {
    atomicOr(err, 1);
    cx = cy = cz = 0.0;
  }
  // s = cp/h, base = floor(s) - 1, t = s - floor(s)   (reading R2)
  double sx = RN_DIV(cx, P.h), sy = RN_DIV(cy, P.h), sz = RN_DIV(cz, P.h);
  double fx = floor(sx), fy = floor(sy), fz = floor(sz);
  tx[e] = RN_SUB(sx, fx);
  ty[e] = RN_SUB(sy, fy);
  tz[e] = RN_SUB(sz, fz);
  ebase[3 * (size_t)e + 0] = (int)fx - 1;
  ebase[3 * (size_t)e + 1] = (int)fy - 1;
  ebase[3 * (size_t)e + 2] = (int)fz - 1;
  ecell[e] = (uint16_t)c;
}

// ------------------------------------------------------------------ B6
__global__ void k_brick_map(int nT, const TileHdr* tiles, const int* blo, const int* bdim,
                            int* bmap) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nT) return;
  int x = tiles[t].bx - blo[0], y = tiles[t].by - blo[1], z = tiles[t].bz - blo[2];
  bmap[((size_t)z * bdim[1] + y) * bdim[0] + x] = t;
}

__device__ inline int bmap_get(const int* bmap, const int* blo, const int* bdim, int bx, int by,
                               int bz) {
  int x = bx - blo[0], y = by - blo[1], z = bz - blo[2];
  if (x < 0 || y < 0 || z < 0 || x >= bdim[0] || y >= bdim[1] || z >= bdim[2]) return -1;
  return bmap[((size_t)z * bdim[1] + y) * bdim[0] + x];
}

// Per tile: stencil box = bounding box of the eval nodes' 4^3 stencils.
__global__ void __launch_bounds__(256) k_tile_box(int nT, TileHdr* tiles, const int32_t* ebase,
                                                  const int* bmap, const int* blo,
                                                  const int* bdim, int* err, int* maxbox) {
  int t = blockIdx.x;
  TileHdr T = tiles[t];
  int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
  for (int e = T.e0 + threadIdx.x; e < T.e1; e += blockDim.x) {
    for (int q = 0; q < 3; ++q) {
      int v = ebase[3 * (size_t)e + q];
      lo[q] = min(lo[q], v);
      hi[q] = max(hi[q], v);
    }
  }
  using BR = cub::BlockReduce<int, 256>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ int res[6];
  for (int q = 0; q < 3; ++q) {
    int a = BR(tmp).Reduce(lo[q], cub::Min());
    __syncthreads();
    int b = BR(tmp).Reduce(hi[q], cub::Max());
    __syncthreads();
    if (threadIdx.x == 0) {
      res[q] = a;
      res[3 + q] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    T.ox = res[0];
    T.oy = res[1];
    T.oz = res[2];
    T.sx = res[3] - res[0] + 4;
    T.sy = res[4] - res[1] + 4;
    T.sz = res[5] - res[2] + 4;
    // padded strides: pick row stride px >= sx and plane stride pxy >= px*sy whose
    // small neighbour offsets fall in distinct double-banks (mod 16), so the
    // sorted stencil gathers of one warp rarely bank-conflict.
    int best = INT_MAX, bpx = T.sx, bpxy = T.sx * T.sy;
    for (int dx = 0; dx < 16; ++dx)
      for (int dz = 0; dz < 16; ++dz) {
        const int px = T.sx + dx, pxy = px * T.sy + dz;
        const int d[9] = {1, px, pxy, px + 1, px - 1, pxy + 1, pxy - 1, pxy + px, pxy - px};
        int score = 0;
        for (int a = 0; a < 9; ++a) {
          if ((d[a] & 15) == 0) score += 16;
          for (int b = a + 1; b < 9; ++b)
            if (((d[a] - d[b]) & 15) == 0) score += 1;
        }
        score = score * 100000 + pxy * T.sz;
        if (score < best) {
          best = score;
          bpx = px;
          bpxy = pxy;
        }
      }
    T.pad[0] = bpx;
    T.pad[1] = bpxy;
    int cells = bpxy * T.sz;
    if (T.sx > kMaxBoxEdge || T.sy > kMaxBoxEdge || T.sz > kMaxBoxEdge || cells > kMaxBoxCells)
      atomicOr(err, 2);
    atomicMax(maxbox, cells);
    T.nbr[0] = bmap_get(bmap, blo, bdim, T.bx + 1, T.by, T.bz);
    T.nbr[1] = bmap_get(bmap, blo, bdim, T.bx - 1, T.by, T.bz);
    T.nbr[2] = bmap_get(bmap, blo, bdim, T.bx, T.by + 1, T.bz);
    T.nbr[3] = bmap_get(bmap, blo, bdim, T.bx, T.by - 1, T.bz);
    T.nbr[4] = bmap_get(bmap, blo, bdim, T.bx, T.by, T.bz + 1);
    T.nbr[5] = bmap_get(bmap, blo, bdim, T.bx, T.by, T.bz - 1);
    tiles[t] = T;
  }
}

// Per eval node: box offset of its stencil base; stencil coverage check (every
// stencil cell must be a source node, i.e. in Sigma_A: StencilEscape otherwise).
__global__ void k_eoff(int nT, const TileHdr* tiles, const int32_t* ebase, const uint16_t* ecell,
                       const uint32_t* tam, const int* bmap, const int* blo, const int* bdim,
                       uint32_t* eoff, int* err) {
  int t = blockIdx.x;
  const TileHdr T = tiles[t];
  for (int e = T.e0 + threadIdx.x; e < T.e1; e += blockDim.x) {
    int b0 = ebase[3 * (size_t)e], b1 = ebase[3 * (size_t)e + 1], b2 = ebase[3 * (size_t)e + 2];
    uint32_t off = (uint32_t)((b0 - T.ox) + T.pad[0] * (b1 - T.oy) + T.pad[1] * (b2 - T.oz));
    eoff[e] = off | ((uint32_t)ecell[e] << 16);  // vb slot = the node's brick cell
    bool ok = true;
    for (int cz = 0; cz < 4 && ok; ++cz)
      for (int cy = 0; cy < 4 && ok; ++cy)
        for (int cx = 0; cx < 4 && ok; ++cx) {
          int i = b0 + cx, j = b1 + cy, k = b2 + cz;
          int s = bmap_get(bmap, blo, bdim, brick_of(i), brick_of(j), brick_of(k));
          if (s < 0) {
            ok = false;
            break;
          }
          int cell = local_of(i) + 8 * local_of(j) + 64 * local_of(k);
          if (!mask_has(tam + (size_t)s * 16, cell)) ok = false;
        }
    if (!ok) atomicOr(err, 4);
  }
}

// ------------------------------------------------------------------ B6b
// Sort each tile's eval nodes by stencil-box offset (bitonic, <= 512 per tile) so
// that lanes of a warp gather overlapping stencils (shared-memory broadcast).
__global__ void __launch_bounds__(512) k_sort_tile(const TileHdr* tiles, double* tx, double* ty,
                                                   double* tz, uint32_t* eoff) {
  __shared__ uint32_t key[512];
  __shared__ double sv[3][512];
  __shared__ uint32_t so[512];
  const TileHdr T = tiles[blockIdx.x];
  const int n = T.e1 - T.e0, t = threadIdx.x;
  if (t < n) {
    const uint32_t eo = eoff[T.e0 + t];
    key[t] = ((eo & 0xffffu) << 9) | (uint32_t)t;
    sv[0][t] = tx[T.e0 + t];
    sv[1][t] = ty[T.e0 + t];
    sv[2][t] = tz[T.e0 + t];
    so[t] = eo;
  } else {
    key[t] = 0xffffffffu;
  }
  __syncthreads();
  for (int size = 2; size <= 512; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const int p = t ^ stride;
      if (p > t) {
        const bool up = (t & size) == 0;
        const uint32_t a = key[t], b = key[p];
        if ((a > b) == up) {
          key[t] = b;
          key[p] = a;
        }
      }
      __syncthreads();
    }
  if (t < n) {
    const int o = key[t] & 511u;
    tx[T.e0 + t] = sv[0][o];
    ty[T.e0 + t] = sv[1][o];
    tz[T.e0 + t] = sv[2][o];
    eoff[T.e0 + t] = so[o];
  }
}

// Box strides for bank spread (both node orders): the dealing needs, per warp,
// items with distinct stencil-base offsets mod 16, so choose the padded strides
// (row stride sx + a, plane stride (sx + a) sy + b, a, b < 16) that make the
// residues of the tile's distinct bases most uniform (largest minimum count, then
// the smallest box), among those no larger than the band's largest box.  Bases
// are decoded from the current offsets; so[] (sorted by offset) is re-encoded.
// Called by all threads of a 512-thread CTA.
__device__ void balance_strides(const TileHdr& T, TileHdr* hdr, uint32_t* so, int n, int boxCap,
                                unsigned long long& best, bool exact = false) {
  const int t = threadIdx.x;
  if (t == 0) best = ~0ull;
  __syncthreads();
  {
    const int px0 = T.pad[0], pxy0 = T.pad[1];
    const int a = t & 15, b = (t >> 4) & 15;
    const int px = T.sx + a, pxy = px * T.sy + b;
    int cnt[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) cnt[r] = 0;
    if (t < 256 && exact) {
      // the gather wavefronts the pair dealing needs with these strides: equal-base
      // groups give c/2 pairs on one address (broadcast) and c % 2 single; per
      // residue r, pair addresses pc[r] and singles sc[r]; pair warps cost
      // >= max(ceil(P/16), max pc), single half-warps >= max(ceil(S/16), max sc)
      int sc[16], P = 0, S = 0;
#pragma unroll
      for (int r = 0; r < 16; ++r) sc[r] = 0;
      for (int i = 0; i < n;) {
        const int o = so[i] & 0xffff;
        int j = i + 1;
        while (j < n && (int)(so[j] & 0xffff) == o) ++j;
        const int dz = o / pxy0, rem = o - dz * pxy0, dy = rem / px0, dx = rem - dy * px0;
        const int r = (dx + px * dy + pxy * dz) & 15, c = j - i;
        if (c >= 2) {
          cnt[r] += (c / 2 + 15) / 16;
          P += c / 2;
        }
        if (c & 1) {
          sc[r]++;
          ++S;
        }
        i = j;
      }
      int mp = 0, ms = 0;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        mp = max(mp, cnt[r]);
        ms = max(ms, sc[r]);
      }
      const int cost = max((P + 15) / 16, mp) + max((S + 15) / 16, ms);
      const unsigned cells = (unsigned)(pxy * T.sz);
      if (cells <= (unsigned)boxCap)
        atomicMin(&best, ((unsigned long long)min(cost, 1023) << 40) | ((unsigned long long)cells << 8) |
                             (unsigned long long)t);
    } else if (t < 256) {
      for (int i = 0; i < n; ++i) {
        const int o = so[i] & 0xffff;
        if (i > 0 && o == (int)(so[i - 1] & 0xffff)) continue;  // distinct bases (sorted input)
        const int dz = o / pxy0, rem = o - dz * pxy0, dy = rem / px0, dx = rem - dy * px0;
        cnt[(dx + px * dy + pxy * dz) & 15]++;
      }
      int mn = 1 << 20;
#pragma unroll
      for (int r = 0; r < 16; ++r) mn = min(mn, cnt[r]);
      const unsigned cells = (unsigned)(pxy * T.sz);
      if (cells <= (unsigned)boxCap)  // never enlarge the band's largest box (smem per CTA)
        atomicMin(&best, ((unsigned long long)(1023 - min(mn, 1023)) << 40) |
                             ((unsigned long long)cells << 8) | (unsigned long long)t);
    }
  }
  __syncthreads();
  if (best != ~0ull) {
    const int bt = (int)(best & 0xff);
    const int px = T.sx + (bt & 15), pxy = px * T.sy + ((bt >> 4) & 15);
    const int px0 = T.pad[0], pxy0 = T.pad[1];
    if (t < n) {
      const int o = so[t] & 0xffff;
      const int dz = o / pxy0, rem = o - dz * pxy0, dy = rem / px0, dx = rem - dy * px0;
      so[t] = (so[t] & 0xffff0000u) | (uint32_t)(dx + px * dy + pxy * dz);
    }
    __syncthreads();
    if (t == 0) {
      hdr->pad[0] = px;
      hdr->pad[1] = pxy;
    }
  }
  __syncthreads();
}

// Deal n items (node indices, sorted by stencil-box offset) into groups of 16
// whose offsets are distinct mod 16 where the residue counts allow it: each group
// takes the head item of the residue class with the most items left among the
// classes it has not used yet (so the classes drain evenly and conflicts are left
// for the last groups only), together with the following items of that class with
// the same offset (one address: a broadcast, free); when every class is used, the
// fullest classes again.  Thread-0 code; out receives the dealt order.
__device__ void deal16(const uint16_t* item, int n, const uint32_t* so, uint16_t* bk, uint16_t* out) {
  int cnt[16], head[16];
  for (int r = 0; r < 16; ++r) cnt[r] = 0;
  for (int i = 0; i < n; ++i) ++cnt[so[item[i]] & 15u];
  int st = 0;
  for (int r = 0; r < 16; ++r) {
    head[r] = st;
    st += cnt[r];
  }
  {
    int pos[16];
    for (int r = 0; r < 16; ++r) pos[r] = head[r];
    for (int i = 0; i < n; ++i) bk[pos[so[item[i]] & 15u]++] = item[i];  // stable: offset order kept
  }
  int left = n, k = 0;
  while (left > 0) {
    int taken = 0;
    uint32_t used = 0;
    while (taken < 16 && left > 0) {
      int best = -1;
      for (int pass = 0; pass < 2 && best < 0; ++pass)
        for (int r = 0; r < 16; ++r)
          if (cnt[r] > 0 && (pass == 1 || !((used >> r) & 1u)) && (best < 0 || cnt[r] > cnt[best])) best = r;
      const uint32_t o = so[bk[head[best]]] & 0xffffu;
      do {
        out[k++] = bk[head[best]++];
        --cnt[best];
        --left;
        ++taken;
      } while (taken < 16 && cnt[best] > 0 && (so[bk[head[best]]] & 0xffffu) == o);
      used |= 1u << best;
    }
  }
}

// ------------------------------------------------------------------ B6c
// Warp order: k_extend_nt gives the tile's nodes 32 at a time to the lanes of a
// warp.  An 8-byte shared-memory load of a warp costs ONE wavefront when every
// adjacent lane pair (2i, 2i+1) reads the same double and the 16 pair addresses
// fall in distinct bank pairs, two otherwise (measured, tools/micro/shfl_vs_lds.cu).
// All 64 gathers of a node are its stencil base + a lane-independent row
// offset, so: nodes of equal base are paired, pairs are dealt 16 to a warp with
// box offsets that are distinct mod 16 or equal (greedy from the base-sorted
// order; when no compatible pair is left, any); the unpaired nodes follow, dealt
// 16 per half-warp by the same rule.
// One CTA per tile, thread 0 plans.
__global__ void __launch_bounds__(512) k_warp_order(TileHdr* tiles, double* tx, double* ty,
                                                    double* tz, uint32_t* eoff, int boxCap, int newdeal) {
  __shared__ double sv[3][512];
  __shared__ uint32_t so[512];
  __shared__ uint16_t perm[512], pfirst[256], single[512], bk[512], dealt[512];
  __shared__ uint8_t pused[512];
  __shared__ int npair, ndup;
  __shared__ unsigned long long best;
  const TileHdr T = tiles[blockIdx.x];
  const int n = T.e1 - T.e0, t = threadIdx.x;
  if (t < n) {
    sv[0][t] = tx[T.e0 + t];
    sv[1][t] = ty[T.e0 + t];
    sv[2][t] = tz[T.e0 + t];
    so[t] = eoff[T.e0 + t];
  }
  balance_strides(T, tiles + blockIdx.x, so, n, boxCap, best, newdeal >= 2);
  if (t == 0) {
    int np = 0, ns = 0;
    for (int i = 0; i < n;) {  // groups of equal base -> pairs + a singleton
      int j = i + 1;
      while (j < n && (so[j] & 0xffffu) == (so[i] & 0xffffu)) ++j;
      int q = i;
      for (; q + 1 < j; q += 2) {
        pfirst[np] = (uint16_t)q;
        pused[np] = 0;
        ++np;
      }
      if (q < j) single[ns++] = (uint16_t)q;
      i = j;
    }
    npair = np;
    // warps of 16 items (a pair on a lane pair; the unpaired nodes that complete the
    // last pair warp on both lanes of a lane pair): pairs first
    int out = 0, taken = 0, nd = 0;
    uint32_t res = 0;
    if (newdeal) {
      deal16(pfirst, np, so, bk, dealt);
      for (int q = 0; q < np; ++q) {
        perm[out++] = dealt[q];
        perm[out++] = (uint16_t)(dealt[q] + 1);
      }
      taken = np & 15;
      for (int q = np - taken; q < np; ++q) res |= 1u << (so[dealt[q]] & 15u);
    } else {
      uint16_t toff[16];
      for (int q = 0; q < np; ++q) pused[q] = 0;
      int first = 0, left = np;
      while (left > 0) {
        for (int pass = 0; pass < 2 && taken < 16; ++pass) {  // compatible first, then any
          for (int q = first; q < np && taken < 16; ++q) {
            if (pused[q]) continue;
            const int node = pfirst[q];
            const uint32_t o = so[node] & 0xffffu, r = o & 15u;
            if (pass == 0) {
              bool ok = !((res >> r) & 1u);
              for (int z = 0; z < taken && !ok; ++z) ok = toff[z] == o;  // same address: broadcast
              if (!ok) continue;
            }
            res |= 1u << r;
            toff[taken++] = (uint16_t)o;
            pused[q] = 1;
            --left;
            perm[out++] = (uint16_t)node;
            perm[out++] = (uint16_t)(node + 1);
          }
        }
        while (first < np && pused[first]) ++first;
        if (taken == 16) {
          taken = 0;
          res = 0;
        }
      }
    }
    for (int q = 0; q < ns; ++q) pused[q] = 0;
    int sleft = ns;
    // the partial last pair warp: completed with unpaired nodes on lane pairs (dup)
    while (taken > 0 && taken < 16 && sleft > 0) {
      int pick = -1;
      for (int q = 0; q < ns && pick < 0; ++q)
        if (!pused[q] && !((res >> (so[single[q]] & 15u)) & 1u)) pick = q;
      for (int q = 0; q < ns && pick < 0; ++q)
        if (!pused[q]) pick = q;
      pused[pick] = 1;
      --sleft;
      res |= 1u << (so[single[pick]] & 15u);
      ++taken;
      ++nd;
      perm[out++] = single[pick];
    }
    // the other unpaired nodes one per lane, 16 per half-warp with distinct residues
    // (16 distinct doubles of a half-warp in distinct bank pairs: one wavefront)
    if (newdeal) {
      int nl = 0;
      for (int q = 0; q < ns; ++q)
        if (!pused[q]) dealt[nl++] = single[q];
      deal16(dealt, nl, so, bk, perm + out);
      out += nl;
    } else {
      taken = 0;
      res = 0;
      int first = 0;
      while (sleft > 0) {
        for (int pass = 0; pass < 2 && taken < 16 && sleft > 0; ++pass) {
          for (int q = first; q < ns && taken < 16; ++q) {
            if (pused[q]) continue;
            const uint32_t r = so[single[q]] & 15u;
            if (pass == 0 && ((res >> r) & 1u)) continue;
            res |= 1u << r;
            ++taken;
            pused[q] = 1;
            --sleft;
            perm[out++] = single[q];
          }
        }
        while (first < ns && pused[first]) ++first;
        if (taken == 16) {
          taken = 0;
          res = 0;
        }
      }
    }
    ndup = nd;
  }
  __syncthreads();
  if (t < n) {
    const int o = perm[t];
    tx[T.e0 + t] = sv[0][o];
    ty[T.e0 + t] = sv[1][o];
    tz[T.e0 + t] = sv[2][o];
    eoff[T.e0 + t] = so[o];
  }
  if (t == 0) {
    tiles[blockIdx.x].np = npair;
    tiles[blockIdx.x].pad2 = ndup;
  }
}

// ------------------------------------------------------------------ B6d
// Item order (the default; k_extend_it in apply.cu): a lane evaluates an ITEM of
// one or two eval nodes with the same stencil base, so each of its 64 shared-memory
// gathers feeds two contractions.  A warp load costs one wavefront per 16 distinct
// doubles in distinct bank pairs (tools/micro/shfl_vs_lds.cu), so
//   * groups of >= 3 equal-base nodes become CHUNKS of 3-4 nodes on a lane pair
//     (2 + 1..2 nodes, one address for both lanes), dealt 16 per warp round with
//     distinct offsets mod 16: one wavefront per gather for up to 64 nodes;
//   * the rest (groups of 1-2, a chunk's remainder of 1-2) are LONE items, one
//     per lane, 16 per half-warp with distinct residues: two wavefronts; rounds
//     of two-node items, then rounds of one-node items (flags 0: the kernel runs
//     the single contraction there).
// Per tile the rounds are words in rnd[T.np .. T.np + T.pad2): bits 0-31 = lane l's
// item has two nodes, bits 32-47 = the round's first node (relative to e0), bits
// 48-53 = lanes in use.  Lane l's item starts at that node + l + popc(bits below l).
// One CTA per tile, thread 0 plans.
constexpr int kMaxRounds = 32;  // per tile: <= 512/3/16 chunk rounds + 512/32 lone rounds
__global__ void __launch_bounds__(512) k_item_order(TileHdr* tiles, double* tx, double* ty,
                                                    double* tz, uint32_t* eoff, uint64_t* rnd,
                                                    int boxCap, int* err) {
  __shared__ double sv[3][512];
  __shared__ uint32_t so[512];
  __shared__ uint16_t perm[512], cstart[512], lstart[512];
  __shared__ uint8_t ccnt[512], lcnt[512], used[512];
  __shared__ unsigned long long best;
  const TileHdr T = tiles[blockIdx.x];
  const int n = T.e1 - T.e0, t = threadIdx.x;
  if (t < n) {
    sv[0][t] = tx[T.e0 + t];
    sv[1][t] = ty[T.e0 + t];
    sv[2][t] = tz[T.e0 + t];
    so[t] = eoff[T.e0 + t];
  }
  balance_strides(T, tiles + blockIdx.x, so, n, boxCap, best);
  if (t == 0) {
    uint64_t* R = rnd + (size_t)blockIdx.x * kMaxRounds;
    int nc = 0, nl = 0;
    for (int i = 0; i < n;) {  // equal-base groups -> chunks of 3-4, lone items of 1-2
      int j = i + 1;
      while (j < n && (so[j] & 0xffffu) == (so[i] & 0xffffu)) ++j;
      int q = i;
      while (j - q >= 3) {
        const int c = min(4, j - q);
        cstart[nc] = (uint16_t)q;
        ccnt[nc++] = (uint8_t)c;
        q += c;
      }
      if (q < j) {
        lstart[nl] = (uint16_t)q;
        lcnt[nl++] = (uint8_t)(j - q);
      }
      i = j;
    }
    int out = 0, nr = 0;
    // chunk rounds: 16 chunks with distinct residues (compatible first, then any)
    for (int q = 0; q < nc; ++q) used[q] = 0;
    int left = nc, first = 0;
    while (left > 0) {
      uint32_t res = 0, flags = 0;
      int taken = 0;
      const int base = out;
      for (int pass = 0; pass < 2 && taken < 16 && left > 0; ++pass)
        for (int q = first; q < nc && taken < 16; ++q) {
          if (used[q]) continue;
          const uint32_t r = so[cstart[q]] & 15u;
          if (pass == 0 && ((res >> r) & 1u)) continue;
          res |= 1u << r;
          used[q] = 1;
          --left;
          const int s0 = cstart[q], c = ccnt[q];
          perm[out++] = (uint16_t)s0;  // lane 2k: two nodes
          perm[out++] = (uint16_t)(s0 + 1);
          flags |= 1u << (2 * taken);
          perm[out++] = (uint16_t)(s0 + 2);  // lane 2k + 1: one or two
          if (c == 4) {
            perm[out++] = (uint16_t)(s0 + 3);
            flags |= 1u << (2 * taken + 1);
          }
          ++taken;
        }
      while (first < nc && used[first]) ++first;
      if (nr < kMaxRounds)
        R[nr] = (uint64_t)flags | ((uint64_t)base << 32) | ((uint64_t)(2 * taken) << 48);
      ++nr;
    }
    // lone rounds, the two-node items first, then the one-node items (rounds of one
    // kind: a round of one-node items runs the single contraction): 16 items per
    // half-warp with distinct residues (a 64-bit warp load is served per half-warp:
    // 16 distinct doubles in distinct bank pairs = one wavefront each)
    for (int q = 0; q < nl; ++q) used[q] = 0;
    for (int kind = 2; kind >= 1; --kind) {
      left = 0;
      for (int q = 0; q < nl; ++q) left += lcnt[q] == kind;
      first = 0;
      while (left > 0) {
        uint32_t flags = 0;
        int taken = 0;
        const int base = out;
        for (int half = 0; half < 2 && left > 0; ++half) {
          uint32_t res = 0;
          int th = 0;
          for (int pass = 0; pass < 2 && th < 16 && left > 0; ++pass)
            for (int q = first; q < nl && th < 16; ++q) {
              if (used[q] || lcnt[q] != kind) continue;
              const uint32_t r = so[lstart[q]] & 15u;
              if (pass == 0 && ((res >> r) & 1u)) continue;
              res |= 1u << r;
              used[q] = 1;
              --left;
              perm[out++] = lstart[q];
              if (kind == 2) {
                perm[out++] = (uint16_t)(lstart[q] + 1);
                flags |= 1u << taken;
              }
              ++taken;
              ++th;
            }
          while (first < nl && (used[first] || lcnt[first] != kind)) ++first;
          if (th < 16) break;  // a partial half ends the round
        }
        if (nr < kMaxRounds)
          R[nr] = (uint64_t)flags | ((uint64_t)base << 32) | ((uint64_t)taken << 48);
        ++nr;
      }
    }
    if (nr > kMaxRounds) atomicOr(err, 8);
    tiles[blockIdx.x].np = blockIdx.x * kMaxRounds;
    tiles[blockIdx.x].pad2 = min(nr, kMaxRounds);
  }
  __syncthreads();
  if (t < n) {
    const int o = perm[t];
    tx[T.e0 + t] = sv[0][o];
    ty[T.e0 + t] = sv[1][o];
    tz[T.e0 + t] = sv[2][o];
    eoff[T.e0 + t] = so[o];
  }
}

// ------------------------------------------------------------------ B7
// Thread per (tile, box row).  Walk the row's x range brick by brick; maximal
// segments of consecutive Sigma_A cells inside one brick row are consecutive in
// band order and become one run (source = band-order index of the first cell).
__global__ void k_rows_per_tile(int nT, const TileHdr* tiles, int64_t* nrows) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nT) nrows[t] = (int64_t)tiles[t].sy * tiles[t].sz + 1;  // + the alignment row
  if (t == 0) nrows[nT] = 0;
}

// Only the cells some stencil of the tile reads are staged: per box row the x
// range is the union of the stencil rows' [b0, b0 + 3] that fall on it.
template <bool WRITE>
__global__ void k_runs(const TileHdr* tiles, const int32_t* ebase, const uint32_t* tam,
                       const int* bmap, const int* blo, const int* bdim, const int64_t* rowbase,
                       int64_t* rowcnt, const int64_t* runstart, uint64_t* runs) {
  __shared__ int xlo[kMaxBoxEdge * kMaxBoxEdge], xhi[kMaxBoxEdge * kMaxBoxEdge];
  __shared__ int tot;
  int t = blockIdx.x;
  const TileHdr T = tiles[t];
  int nrows = T.sy * T.sz;
  for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
    xlo[r] = INT_MAX;
    xhi[r] = INT_MIN;
  }
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  for (int e = T.e0 + threadIdx.x; e < T.e1; e += blockDim.x) {
    const int b0 = ebase[3 * (size_t)e], b1 = ebase[3 * (size_t)e + 1] - T.oy,
              b2 = ebase[3 * (size_t)e + 2] - T.oz;
    for (int dz = 0; dz < 4; ++dz)
      for (int dy = 0; dy < 4; ++dy) {
        const int r = (b1 + dy) + T.sy * (b2 + dz);
        atomicMin(&xlo[r], b0);
        atomicMax(&xhi[r], b0 + 4);
      }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
    int y = T.oy + r % T.sy, z = T.oz + r / T.sy;
    int by = brick_of(y), bz = brick_of(z), ly = local_of(y), lz = local_of(z);
    int64_t gi = rowbase[t] + r;
    int64_t out = WRITE ? runstart[gi] : 0;
    int64_t n = 0;
    int x = xlo[r], xe = xhi[r];  // empty row: x = INT_MAX > xe
    while (x < xe) {
      int bx = brick_of(x);
      int xend = min(xe, bx * 8 + 8);
      int s = bmap_get(bmap, blo, bdim, bx, by, bz);
      if (s >= 0) {
        const uint32_t* m = tam + (size_t)s * 16;
        int q = local_of(x), lxe = xend - bx * 8;
        while (q < lxe) {
          if (!mask_has(m, q + 8 * ly + 64 * lz)) {
            ++q;
            continue;
          }
          int q0 = q;
          while (q < lxe && mask_has(m, q + 8 * ly + 64 * lz)) ++q;
          if (WRITE) {
            uint32_t src = (uint32_t)(tiles[s].a0 + mask_rank(m, q0 + 8 * ly + 64 * lz));
            uint32_t dst = (uint32_t)((bx * 8 + q0 - T.ox) + T.pad[0] * (y - T.oy) + T.pad[1] * (z - T.oz));
            runs[out + n] = pack_run(src, dst, (uint32_t)(q - q0));
          }
          ++n;
        }
      }
      x = xend;
    }
    if (!WRITE) {
      rowcnt[gi] = n;
      atomicAdd(&tot, (int)n);
    }
  }
  // alignment row: one empty run when the tile has an odd number of runs, so
  // every tile's run range starts 16-byte aligned (bulk copies)
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t gi = rowbase[t] + nrows;
    if (WRITE) {
      if (rowbase[t + 1] - rowbase[t] == nrows + 1 && runstart[gi + 1] > runstart[gi])
        runs[runstart[gi]] = 0ull;
    } else {
      rowcnt[gi] = tot & 1;
    }
  }
}

__global__ void k_set_run_ranges(int nT, TileHdr* tiles, const int64_t* rowbase,
                                 const int64_t* runstart) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nT) return;
  tiles[t].r0 = (int32_t)runstart[rowbase[t]];
  tiles[t].r1 = (int32_t)runstart[rowbase[t + 1]];
}

__global__ void k_run_offsets(int nT, const TileHdr* tiles, int* beg, int* end) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nT) return;
  beg[t] = tiles[t].r0;
  end[t] = tiles[t].r1;
}

// eval ranges start at multiples of 4 nodes (16-byte aligned for bulk copies)
__global__ void k_round4(int nb, const int* ne, int* ne4) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) ne4[b] = (ne[b] + 3) & ~3;
  if (b == 0) ne4[nb] = 0;
}

__global__ void k_max_box(int nT, const TileHdr* tiles, int* mx) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nT) atomicMax(mx, tiles[t].pad[1] * tiles[t].sz);
}

__global__ void k_flags(int nb, const int* ne, int* flag) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) flag[b] = ne[b] > 0 ? 1 : 0;
  if (b == 0) flag[nb] = 0;
}

// ------------------------------------------------------------------ F (fused-apply experiment)
// For the single-kernel apply (apply.cu k_apply_fused): every tile also evaluates
// E u at its HALO nodes — the eval nodes of face-neighbour tiles that are 6-neighbours
// of its own active nodes — so no E u crosses HBM.  Its box must cover the halo
// nodes' stencils too (the "fused box"); the own nodes keep their order (pairs).
// Bases are decoded from the final box offsets (the eval order was permuted).
__device__ inline void decode_base(const TileHdr& T, uint32_t eo, int* b) {
  const int o = (int)(eo & 0xffffu);
  const int dz = o / T.pad[1], rem = o - dz * T.pad[1], dy = rem / T.pad[0], dx = rem - dy * T.pad[0];
  b[0] = T.ox + dx;
  b[1] = T.oy + dy;
  b[2] = T.oz + dz;
}

// cell -> local eval index of every tile (0xffff: not an eval cell)
__global__ void k_fz_cmap(const TileHdr* tiles, const uint32_t* eoff, uint16_t* cmap) {
  const int t = blockIdx.x;
  const TileHdr T = tiles[t];
  for (int c = threadIdx.x; c < 512; c += blockDim.x) cmap[(size_t)t * 512 + c] = 0xffffu;
  __syncthreads();
  for (int e = T.e0 + threadIdx.x; e < T.e1; e += blockDim.x)
    cmap[(size_t)t * 512 + (eoff[e] >> 16)] = (uint16_t)(e - T.e0);
}

// halo nodes of tile t: face f, face cell (i, j): own boundary cell active and the
// neighbour's facing cell an eval cell.  WRITE = false counts, true fills.
template <bool WRITE>
__global__ void k_fz_halo(const TileHdr* tiles, const uint32_t* tam, const uint16_t* cmap, int* cnt,
                          const int* hstart, uint64_t* halo) {
  const int t = blockIdx.x, q = threadIdx.x;  // 384 threads: f = q / 64
  __shared__ int n;
  if (q == 0) n = 0;
  __syncthreads();
  const TileHdr T = tiles[t];
  const int f = q >> 6, i = q & 7, j = (q >> 3) & 7;
  const int src = T.nbr[f];
  bool take = false;
  int c = 0, h = 0;
  if (src >= 0) {
    const int axis = f >> 1, plus = (f & 1) == 0;
    const int in = plus ? 0 : 7, me = plus ? 7 : 0, out = plus ? 8 : -1;
    int co;
    if (axis == 0) { c = in + 8 * i + 64 * j; co = me + 8 * i + 64 * j; h = (out + 1) + 10 * (i + 1) + 100 * (j + 1); }
    else if (axis == 1) { c = i + 8 * in + 64 * j; co = i + 8 * me + 64 * j; h = (i + 1) + 10 * (out + 1) + 100 * (j + 1); }
    else { c = i + 8 * j + 64 * in; co = i + 8 * j + 64 * me; h = (i + 1) + 10 * (j + 1) + 100 * (out + 1); }
    take = mask_has(tam + (size_t)t * 16, co) && cmap[(size_t)src * 512 + c] != 0xffffu;
  }
  if (take) {
    const int k = atomicAdd(&n, 1);
    if (WRITE) {
      const uint32_t e = (uint32_t)(tiles[src].e0 + cmap[(size_t)src * 512 + c]);
      halo[hstart[t] + k] = (uint64_t)e | ((uint64_t)h << 48);
    }
  }
  __syncthreads();
  if (!WRITE && q == 0) cnt[t] = n;
}

// the union of own and halo stencil bases per tile into ub (tile t at e0 + hstart[t] ..),
// and the temp header ft with that range; bbox + strides of the fused box
__global__ void __launch_bounds__(256) k_fz_box(int nT, const TileHdr* tiles, const uint32_t* eoff,
                                                const int* hstart, const uint64_t* halo, int32_t* ub,
                                                TileHdr* ft, int* err, int* maxbox) {
  const int t = blockIdx.x;
  TileHdr T = tiles[t];
  const int ne = T.e1 - T.e0, h0 = hstart[t], nh = hstart[t + 1] - h0, u0 = T.e0 + h0;
  int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
  for (int k = threadIdx.x; k < ne + nh; k += blockDim.x) {
    int b[3];
    if (k < ne) {
      decode_base(T, eoff[T.e0 + k], b);
    } else {
      const uint64_t hv = halo[h0 + k - ne];
      const uint32_t e = (uint32_t)hv;
      // the node's own tile: found through the eval ranges (binary search)
      int l = 0, r = nT - 1;
      while (l < r) {
        const int m = (l + r + 1) >> 1;
        if (tiles[m].e0 <= (int)e) l = m; else r = m - 1;
      }
      decode_base(tiles[l], eoff[e], b);
    }
    for (int q = 0; q < 3; ++q) {
      ub[3 * (size_t)(u0 + k) + q] = b[q];
      lo[q] = min(lo[q], b[q]);
      hi[q] = max(hi[q], b[q]);
    }
  }
  using BR = cub::BlockReduce<int, 256>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ int res[6];
  for (int q = 0; q < 3; ++q) {
    const int a = BR(tmp).Reduce(lo[q], cub::Min());
    __syncthreads();
    const int b = BR(tmp).Reduce(hi[q], cub::Max());
    __syncthreads();
    if (threadIdx.x == 0) {
      res[q] = a;
      res[3 + q] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    T.ox = res[0];
    T.oy = res[1];
    T.oz = res[2];
    T.sx = res[3] - res[0] + 4;
    T.sy = res[4] - res[1] + 4;
    T.sz = res[5] - res[2] + 4;
    // the same stride rule as k_tile_box (small neighbour offsets in distinct banks)
    int best = INT_MAX, bpx = T.sx, bpxy = T.sx * T.sy;
    for (int dx = 0; dx < 16; ++dx)
      for (int dz = 0; dz < 16; ++dz) {
        const int px = T.sx + dx, pxy = px * T.sy + dz;
        const int d[9] = {1, px, pxy, px + 1, px - 1, pxy + 1, pxy - 1, pxy + px, pxy - px};
        int score = 0;
        for (int a = 0; a < 9; ++a) {
          if ((d[a] & 15) == 0) score += 16;
          for (int b = a + 1; b < 9; ++b)
            if (((d[a] - d[b]) & 15) == 0) score += 1;
        }
        score = score * 100000 + pxy * T.sz;
        if (score < best) {
          best = score;
          bpx = px;
          bpxy = pxy;
        }
      }
    T.pad[0] = bpx;
    T.pad[1] = bpxy;
    const int cells = bpxy * T.sz;
    if (T.sx > kMaxBoxEdge || T.sy > kMaxBoxEdge || T.sz > kMaxBoxEdge || cells > kMaxBoxCells) atomicOr(err, 1);
    atomicMax(maxbox, cells);
    T.e0 = u0;  // the temp header's node range: into ub
    T.e1 = u0 + ne + nh;
    ft[t] = T;
  }
}

// fused-box offsets of the own nodes and the halo nodes
__global__ void k_fz_offsets(const TileHdr* tiles, const TileHdr* ft, const int* hstart, const int32_t* ub,
                             const uint32_t* eoff, uint32_t* fzeoff, uint64_t* halo) {
  const int t = blockIdx.x;
  const TileHdr T = tiles[t], F = ft[t];
  const int ne = T.e1 - T.e0, h0 = hstart[t], nh = hstart[t + 1] - h0;
  for (int k = threadIdx.x; k < ne + nh; k += blockDim.x) {
    const int32_t* b = ub + 3 * (size_t)(F.e0 + k);
    const uint32_t off = (uint32_t)((b[0] - F.ox) + F.pad[0] * (b[1] - F.oy) + F.pad[1] * (b[2] - F.oz));
    if (k < ne) fzeoff[T.e0 + k] = off | (eoff[T.e0 + k] & 0xffff0000u);
    else halo[h0 + k - ne] |= (uint64_t)off << 32;
  }
}

// ------------------------------------------------------------------ host helpers
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() {
    return (T*)p;
  }
};

// non-owning view with the DevBuf accessor
template <class E>
struct PtrView {
  E* p;
  template <class T>
  T* as() {
    return (T*)p;
  }
};

template <class T>
int dalloc(DevBuf& b, size_t n, const char* what) {
  cudaError_t e = cudaMalloc(&b.p, std::max<size_t>(n, 1) * sizeof(T));
  if (e != cudaSuccess) return fail(CPM_ERR_NOMEM, std::string("cudaMalloc failed for ") + what);
  return CPM_OK;
}

template <class T>
int dalloc_owned(T** p, size_t n, int64_t* bytes, const char* what) {
  cudaError_t e = cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T));
  if (e != cudaSuccess) return fail(CPM_ERR_NOMEM, std::string("cudaMalloc failed for ") + what);
  *bytes += (int64_t)(std::max<size_t>(n, 1) * sizeof(T));
  return CPM_OK;
}

template <class T>
int exclusive_sum(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  CPM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  DevBuf tb;
  CPM_TRY(dalloc<char>(tb, tmp, "scan temp"));
  CPM_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, tmp, in, out, n, s));
  return CPM_OK;
}

template <class T>
int read_back(const T* dptr, T* hval, cudaStream_t s) {
  CPM_CUDA(cudaMemcpyAsync(hval, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  return CPM_OK;
}

inline int grid_for(int64_t n, int bs) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + bs - 1) / bs, 1 << 30)); }

__global__ void k_fz_restore(int nT, const TileHdr* tiles, TileHdr* ft) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nT) {  // back to the eval-node range (the runs were built over the ub range)
    ft[t].e0 = tiles[t].e0;
    ft[t].e1 = tiles[t].e1;
  }
}

int build_fused(cpm_band* B, const int* bmap, const int* dblo, const int* dbdim, cudaStream_t s) {
  const int nT = B->nT;
  DevBuf cmap, cnt, hst, ftb, ub, err;
  CPM_TRY(dalloc<uint16_t>(cmap, (size_t)nT * 512, "fz cmap"));
  CPM_TRY(dalloc<int>(cnt, nT + 1, "fz cnt"));
  CPM_TRY(dalloc<int>(err, 2, "fz err"));
  CPM_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (nT + 1), s));
  CPM_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int) * 2, s));
  k_fz_cmap<<<nT, 256, 0, s>>>(B->tiles, B->eoff, cmap.as<uint16_t>());
  k_fz_halo<false><<<nT, 384, 0, s>>>(B->tiles, B->amask, cmap.as<uint16_t>(), cnt.as<int>(), nullptr, nullptr);
  CPM_TRY(dalloc_owned(&B->fzH, (size_t)nT + 1, &B->bytes, "fz hstart"));
  CPM_TRY(exclusive_sum(cnt.as<int>(), B->fzH, nT + 1, s));
  int nH = 0;
  CPM_TRY(read_back(B->fzH + nT, &nH, s));
  B->fzNHalo = nH;
  CPM_TRY(dalloc_owned(&B->fzHalo, (size_t)std::max(nH, 1), &B->bytes, "fz halo"));
  k_fz_halo<true><<<nT, 384, 0, s>>>(B->tiles, B->amask, cmap.as<uint16_t>(), nullptr, B->fzH, B->fzHalo);
  // note: the halo list order inside a tile is atomic-order (any order is correct)
  CPM_TRY(dalloc<TileHdr>(ftb, nT, "fz tiles"));
  CPM_TRY(dalloc<int32_t>(ub, 3 * ((size_t)B->nE + 8 + (size_t)nH), "fz bases"));
  k_fz_box<<<nT, 256, 0, s>>>(nT, B->tiles, B->eoff, B->fzH, B->fzHalo, ub.as<int32_t>(), ftb.as<TileHdr>(),
                              err.as<int>(), err.as<int>() + 1);
  CPM_TRY(dalloc_owned(&B->fzEoff, (size_t)B->nE + 8, &B->bytes, "fz eoff"));
  k_fz_offsets<<<nT, 256, 0, s>>>(B->tiles, ftb.as<TileHdr>(), B->fzH, ub.as<int32_t>(), B->eoff, B->fzEoff,
                                  B->fzHalo);
  int herr[2] = {0, 0};
  CPM_CUDA(cudaMemcpyAsync(herr, err.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  if (herr[0]) return fail(CPM_ERR_LIMIT, "fused apply: a fused stencil box exceeds the limit");
  B->fzMaxBox = herr[1];
  // fill runs of the fused boxes (k_runs over the own + halo bases)
  DevBuf nrows, rowbase, rowcnt, runstart;
  CPM_TRY(dalloc<int64_t>(nrows, nT + 1, "fz nrows"));
  CPM_TRY(dalloc<int64_t>(rowbase, nT + 1, "fz rowbase"));
  k_rows_per_tile<<<grid_for(nT + 1, 256), 256, 0, s>>>(nT, ftb.as<TileHdr>(), nrows.as<int64_t>());
  CPM_TRY(exclusive_sum(nrows.as<int64_t>(), rowbase.as<int64_t>(), nT + 1, s));
  int64_t totRows = 0;
  CPM_TRY(read_back(rowbase.as<int64_t>() + nT, &totRows, s));
  CPM_TRY(dalloc<int64_t>(rowcnt, totRows + 1, "fz rowcnt"));
  CPM_TRY(dalloc<int64_t>(runstart, totRows + 1, "fz runstart"));
  CPM_CUDA(cudaMemsetAsync(rowcnt.p, 0, (totRows + 1) * sizeof(int64_t), s));
  k_runs<false><<<nT, 128, 0, s>>>(ftb.as<TileHdr>(), ub.as<int32_t>(), B->amask, bmap, dblo, dbdim,
                                   rowbase.as<int64_t>(), rowcnt.as<int64_t>(), nullptr, nullptr);
  CPM_TRY(exclusive_sum(rowcnt.as<int64_t>(), runstart.as<int64_t>(), totRows + 1, s));
  int64_t totRuns = 0;
  CPM_TRY(read_back(runstart.as<int64_t>() + totRows, &totRuns, s));
  CPM_TRY(dalloc_owned(&B->fzRuns, (size_t)totRuns + 2, &B->bytes, "fz runs"));
  k_runs<true><<<nT, 128, 0, s>>>(ftb.as<TileHdr>(), ub.as<int32_t>(), B->amask, bmap, dblo, dbdim,
                                  rowbase.as<int64_t>(), rowcnt.as<int64_t>(), runstart.as<int64_t>(), B->fzRuns);
  k_set_run_ranges<<<grid_for(nT, 256), 256, 0, s>>>(nT, ftb.as<TileHdr>(), rowbase.as<int64_t>(),
                                                      runstart.as<int64_t>());
  B->fzNRuns = totRuns;
  k_fz_restore<<<grid_for(nT, 256), 256, 0, s>>>(nT, B->tiles, ftb.as<TileHdr>());
  CPM_TRY(dalloc_owned(&B->fzT, (size_t)nT, &B->bytes, "fz tiles"));
  CPM_CUDA(cudaMemcpyAsync(B->fzT, ftb.p, sizeof(TileHdr) * nT, cudaMemcpyDeviceToDevice, s));
  CPM_CUDA(cudaGetLastError());
  CPM_CUDA(cudaStreamSynchronize(s));
  return CPM_OK;
}

}  // namespace

void free_workspace(Workspace* w);

void free_band(cpm_band* b) {
  if (!b) return;
  if (b->ws) free_workspace(b->ws);
  if (b->as) {
    cpm_band::AsyncStage* a = b->as;
    if (a->out) cudaStreamSynchronize(a->out);
    for (int q = 0; q < 2; ++q) {
      if (a->u[q]) cudaFree(a->u[q]);
      if (a->y[q]) cudaFree(a->y[q]);
      for (cudaEvent_t e : {a->ein[q], a->ek[q], a->eout[q]})
        if (e) cudaEventDestroy(e);
    }
    if (a->in) cudaStreamDestroy(a->in);
    if (a->out) cudaStreamDestroy(a->out);
    delete a;
  }
  if (b->owns) {
    void* ptrs[] = {b->tiles, b->tx,      b->ty,      b->tz,    b->eoff, b->acell,
                    b->aijk,  b->gijk,    b->runs,    b->vb,    b->dstage0, b->dstage1,
                    b->amask, b->bmap,    b->rnd,     b->fzT,     b->fzH,   b->fzHalo, b->fzEoff, b->fzRuns};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  } else {  // sub-band: owns only its own tiles/runs/acell/vb
    void* ptrs[] = {b->tiles, b->runs, b->vb, b->acell, b->dstage0, b->dstage1};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
  delete b;
}

int build_band(const cpm_surface* surf, double h, int p, double L, cudaStream_t s,
               cpm_band** out) {
  if (!surf || !out) return fail(CPM_ERR_ARG, "cpm_build_band: null argument");
  *out = nullptr;
  if (p != 3) return fail(CPM_ERR_ARG, "cpm_build_band: only p = 3 (tricubic) is implemented");
  if (!(h > 0.0) || !(L > 0.0)) return fail(CPM_ERR_ARG, "cpm_build_band: h and L must be > 0");
  if (surf->kind != CPM_SURF_SPHERE && surf->kind != CPM_SURF_TORUS)
    return fail(CPM_ERR_ARG, "cpm_build_band: unknown surface kind");
  if (surf->kind == CPM_SURF_SPHERE && !(surf->param[0] > 0.0))
    return fail(CPM_ERR_ARG, "cpm_build_band: sphere radius must be > 0");
  if (surf->kind == CPM_SURF_TORUS && !(surf->param[0] > surf->param[1] && surf->param[1] > 0.0))
    return fail(CPM_ERR_ARG, "cpm_build_band: torus needs R > r > 0");

  BuildParams P;
  P.s.kind = surf->kind;
  for (int q = 0; q < 4; ++q) P.s.p[q] = surf->param[q];
  P.h = h;
  P.lam = sqrt(17.0) * h;  // reading R1
  P.M = (int)llround(L / h);
  P.slack = 1e-9 * h;
  if (P.M > (1 << 18)) return fail(CPM_ERR_LIMIT, "cpm_build_band: L/h too large (> 2^18)");
  double ex, ez;
  if (surf->kind == CPM_SURF_SPHERE) {
    ex = ez = surf->param[0] + P.lam + 2 * h;
  } else {
    ex = surf->param[0] + surf->param[1] + P.lam + 2 * h;
    ez = surf->param[1] + P.lam + 2 * h;
  }
  int ilo[3], ihi[3];
  double e3[3] = {ex, ex, ez};
  for (int q = 0; q < 3; ++q) {
    ilo[q] = std::max(-P.M - 1, (int)floor(-e3[q] / h) - 1);
    ihi[q] = std::min(P.M + 1, (int)ceil(e3[q] / h) + 1);
    P.blo[q] = brick_of(ilo[q]);
    P.bdim[q] = brick_of(ihi[q]) - P.blo[q] + 1;
  }
  int64_t nbox = (int64_t)P.bdim[0] * P.bdim[1] * P.bdim[2];

  // B1 candidates
  DevBuf keys, cnt;
  CPM_TRY(dalloc<uint64_t>(keys, nbox, "brick keys"));
  CPM_TRY(dalloc<int>(cnt, 1, "count"));
  CPM_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), s));
  k_brick_candidates<<<grid_for(nbox, 256), 256, 0, s>>>(P, keys.as<uint64_t>(), cnt.as<int>());
  count_launch();
  CPM_CUDA(cudaGetLastError());
  int nb = 0;
  CPM_TRY(read_back(cnt.as<int>(), &nb, s));
  if (nb == 0) return fail(CPM_ERR_GEOM, "cpm_build_band: empty band (surface outside the box?)");

  // B2 sort by Morton code
  DevBuf keys2;
  CPM_TRY(dalloc<uint64_t>(keys2, nb, "sorted keys"));
  {
    size_t tmp = 0;
    CPM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                            nb, 0, 51, s));
    DevBuf tb;
    CPM_TRY(dalloc<char>(tb, tmp, "sort temp"));
    CPM_CUDA(cub::DeviceRadixSort::SortKeys(tb.p, tmp, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                            nb, 0, 51, s));
  }

  // B3 classify
  DevBuf amask, gmask, na, ng, ne;
  CPM_TRY(dalloc<uint32_t>(amask, (size_t)nb * 16, "amask"));
  CPM_TRY(dalloc<uint32_t>(gmask, (size_t)nb * 16, "gmask"));
  CPM_TRY(dalloc<int>(na, nb + 1, "na"));
  CPM_TRY(dalloc<int>(ng, nb + 1, "ng"));
  CPM_TRY(dalloc<int>(ne, nb + 1, "ne"));
  CPM_CUDA(cudaMemsetAsync(na.p, 0, (nb + 1) * sizeof(int), s));
  CPM_CUDA(cudaMemsetAsync(ng.p, 0, (nb + 1) * sizeof(int), s));
  CPM_CUDA(cudaMemsetAsync(ne.p, 0, (nb + 1) * sizeof(int), s));
  k_classify<<<nb, 512, 0, s>>>(P, keys2.as<uint64_t>(), amask.as<uint32_t>(), gmask.as<uint32_t>(),
                                na.as<int>(), ng.as<int>(), ne.as<int>());
  count_launch();
  CPM_CUDA(cudaGetLastError());

  // B4 scans
  DevBuf astart, gstart, estart, flag, tslot;
  CPM_TRY(dalloc<int>(astart, nb + 1, "astart"));
  CPM_TRY(dalloc<int>(gstart, nb + 1, "gstart"));
  CPM_TRY(dalloc<int>(estart, nb + 1, "estart"));
  CPM_TRY(dalloc<int>(flag, nb + 1, "flag"));
  CPM_TRY(dalloc<int>(tslot, nb + 1, "tslot"));
  CPM_TRY(exclusive_sum(na.as<int>(), astart.as<int>(), nb + 1, s));
  CPM_TRY(exclusive_sum(ng.as<int>(), gstart.as<int>(), nb + 1, s));
  {
    DevBuf ne4;
    CPM_TRY(dalloc<int>(ne4, nb + 1, "ne4"));
    k_round4<<<grid_for(nb + 1, 256), 256, 0, s>>>(nb, ne.as<int>(), ne4.as<int>());
    count_launch();
    CPM_TRY(exclusive_sum(ne4.as<int>(), estart.as<int>(), nb + 1, s));
  }
  k_flags<<<grid_for(nb, 256), 256, 0, s>>>(nb, ne.as<int>(), flag.as<int>());
  count_launch();
  CPM_TRY(exclusive_sum(flag.as<int>(), tslot.as<int>(), nb + 1, s));
  int totA = 0, totG = 0, totE = 0, totT = 0;
  CPM_TRY(read_back(astart.as<int>() + nb, &totA, s));
  CPM_TRY(read_back(gstart.as<int>() + nb, &totG, s));
  CPM_TRY(read_back(estart.as<int>() + nb, &totE, s));
  CPM_TRY(read_back(tslot.as<int>() + nb, &totT, s));
  if (totA == 0) return fail(CPM_ERR_GEOM, "cpm_build_band: no active nodes");

  cpm_band* B = new cpm_band();
  std::unique_ptr<cpm_band, void (*)(cpm_band*)> guard(B, free_band);
  B->surf = P.s;
  B->h = h;
  B->lam = P.lam;
  B->L = L;
  B->M = P.M;
  B->nA = totA;
  B->nG = totG;
  B->nE = totE;
  B->nT = totT;
  B->nOwned = totA;
  for (int q = 0; q < 3; ++q) {
    B->ilo[q] = ilo[q];
    B->ihi[q] = ihi[q];
  }
  DevBuf tgm, tgstart;
  CPM_TRY(dalloc_owned(&B->tiles, totT, &B->bytes, "tiles"));
  CPM_TRY(dalloc_owned(&B->amask, (size_t)totT * 16, &B->bytes, "tile amask"));
  PtrView<uint32_t> tam{B->amask};
  CPM_TRY(dalloc<uint32_t>(tgm, (size_t)totT * 16, "tile gmask"));
  CPM_TRY(dalloc<int>(tgstart, totT, "tile gstart"));
  k_compact_tiles<<<grid_for(nb, 256), 256, 0, s>>>(
      nb, ne.as<int>(), tslot.as<int>(), na.as<int>(), ng.as<int>(), astart.as<int>(),
      gstart.as<int>(), estart.as<int>(), keys2.as<uint64_t>(), amask.as<uint32_t>(),
      gmask.as<uint32_t>(), B->tiles, tam.as<uint32_t>(), tgm.as<uint32_t>(), tgstart.as<int>());
  count_launch();
  CPM_CUDA(cudaGetLastError());

  // B5 per-node data
  DevBuf ebase, ecell, err;
  CPM_TRY(dalloc_owned(&B->aijk, 3 * (size_t)totA, &B->bytes, "aijk"));
  CPM_TRY(dalloc_owned(&B->gijk, 3 * (size_t)std::max(totG, 1), &B->bytes, "gijk"));
  CPM_TRY(dalloc_owned(&B->acell, totA, &B->bytes, "acell"));
  CPM_TRY(dalloc_owned(&B->tx, (size_t)totE + 8, &B->bytes, "tx"));
  CPM_TRY(dalloc_owned(&B->ty, (size_t)totE + 8, &B->bytes, "ty"));
  CPM_TRY(dalloc_owned(&B->tz, (size_t)totE + 8, &B->bytes, "tz"));
  CPM_TRY(dalloc_owned(&B->eoff, (size_t)totE + 8, &B->bytes, "eoff"));
  CPM_TRY(dalloc<int32_t>(ebase, 3 * (size_t)totE, "ebase"));
  CPM_TRY(dalloc<uint16_t>(ecell, totE, "ecell"));
  CPM_TRY(dalloc<int>(err, 2, "err"));
  CPM_CUDA(cudaMemsetAsync(err.p, 0, 2 * sizeof(int), s));
  k_node_data<<<totT, 512, 0, s>>>(P, B->tiles, tam.as<uint32_t>(), tgm.as<uint32_t>(),
                                   tgstart.as<int>(), B->aijk, B->gijk, B->acell, B->tx, B->ty,
                                   B->tz, ebase.as<int32_t>(), ecell.as<uint16_t>(), err.as<int>());
  count_launch();
  CPM_CUDA(cudaGetLastError());

  // B6 brick map, boxes, offsets, coverage
  DevBuf dblo, dbdim;
  CPM_TRY(dalloc_owned(&B->bmap, nbox, &B->bytes, "brick map"));
  for (int q = 0; q < 3; ++q) {
    B->blo[q] = P.blo[q];
    B->bdim[q] = P.bdim[q];
  }
  PtrView<int> bmap{B->bmap};
  CPM_TRY(dalloc<int>(dblo, 3, "blo"));
  CPM_TRY(dalloc<int>(dbdim, 3, "bdim"));
  CPM_CUDA(cudaMemcpyAsync(dblo.p, P.blo, 3 * sizeof(int), cudaMemcpyHostToDevice, s));
  CPM_CUDA(cudaMemcpyAsync(dbdim.p, P.bdim, 3 * sizeof(int), cudaMemcpyHostToDevice, s));
  CPM_CUDA(cudaMemsetAsync(bmap.p, 0xff, nbox * sizeof(int), s));
  k_brick_map<<<grid_for(totT, 256), 256, 0, s>>>(totT, B->tiles, dblo.as<int>(), dbdim.as<int>(),
                                                   bmap.as<int>());
  count_launch();
  k_tile_box<<<totT, 256, 0, s>>>(totT, B->tiles, ebase.as<int32_t>(), bmap.as<int>(),
                                  dblo.as<int>(), dbdim.as<int>(), err.as<int>(),
                                  err.as<int>() + 1);
  count_launch();
  k_eoff<<<totT, 128, 0, s>>>(totT, B->tiles, ebase.as<int32_t>(), ecell.as<uint16_t>(),
                              tam.as<uint32_t>(), bmap.as<int>(), dblo.as<int>(), dbdim.as<int>(),
                              B->eoff, err.as<int>());
  count_launch();
  CPM_CUDA(cudaGetLastError());
  int herr[2] = {0, 0};
  CPM_CUDA(cudaMemcpyAsync(herr, err.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  if (herr[0] & 1)
    return fail(CPM_ERR_GEOM,
                "cpm_build_band: closest point undefined at a band/ghost node (lambda + h exceeds "
                "the surface's reach, PAPER.md:62)");
  if (herr[0] & 2) return fail(CPM_ERR_LIMIT, "cpm_build_band: a tile's stencil box exceeds the limit");
  if (herr[0] & 4)
    return fail(CPM_ERR_GEOM, "cpm_build_band: StencilEscape — an interpolation stencil leaves Sigma_A");
  B->maxBox = herr[1];
  k_sort_tile<<<totT, 512, 0, s>>>(B->tiles, B->tx, B->ty, B->tz, B->eoff);
  count_launch();
  CPM_CUDA(cudaGetLastError());

  // B6c/B6d node order for the extend: items (default) or pairs (CPM_ITEMS=0, the
  // round-1 kernel k_extend_nt, kept for A/B)
  B->itemOrder = (getenv("CPM_ITEMS") && *getenv("CPM_ITEMS") == '1') &&
                 !(getenv("CPM_FUSED") && *getenv("CPM_FUSED") == '1');  // the fused kernel uses pairs
  if (B->itemOrder) {
    CPM_TRY(dalloc_owned(&B->rnd, (size_t)totT * kMaxRounds, &B->bytes, "item rounds"));
    k_item_order<<<totT, 512, 0, s>>>(B->tiles, B->tx, B->ty, B->tz, B->eoff, B->rnd, B->maxBox,
                                      err.as<int>());
    count_launch();
    CPM_CUDA(cudaGetLastError());
    int herr2 = 0;
    CPM_CUDA(cudaMemcpyAsync(&herr2, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CPM_CUDA(cudaStreamSynchronize(s));
    if (herr2 & 8) return fail(CPM_ERR_LIMIT, "cpm_build_band: a tile needs more than 32 item rounds");
  } else {
    // CPM_DEAL=0: the round-1 greedy dealing and residue balance; 1: class-draining
    // dealing; 2 (default): that dealing with strides chosen by its wavefront bound
    // (restricting the row stride to 4 mod 8 for a conflict-free fill of consecutive
    // rows was measured: fill wavefronts 3.15M -> 2.86M, gathers 15.6M -> 16.1M, +0.8 us)
    const int newdeal = getenv("CPM_DEAL") ? atoi(getenv("CPM_DEAL")) : 2;
    k_warp_order<<<totT, 512, 0, s>>>(B->tiles, B->tx, B->ty, B->tz, B->eoff, B->maxBox, newdeal);
    count_launch();
    CPM_CUDA(cudaGetLastError());
  }
  {  // the strides may have changed: largest box again
    DevBuf mb;
    CPM_TRY(dalloc<int>(mb, 1, "max box"));
    CPM_CUDA(cudaMemsetAsync(mb.p, 0, sizeof(int), s));
    k_max_box<<<grid_for(totT, 256), 256, 0, s>>>(totT, B->tiles, mb.as<int>());
    count_launch();
    CPM_CUDA(cudaMemcpyAsync(&B->maxBox, mb.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CPM_CUDA(cudaStreamSynchronize(s));
  }

  // B7 fill runs
  DevBuf nrows, rowbase, rowcnt, runstart;
  CPM_TRY(dalloc<int64_t>(nrows, totT + 1, "nrows"));
  CPM_TRY(dalloc<int64_t>(rowbase, totT + 1, "rowbase"));
  k_rows_per_tile<<<grid_for(totT + 1, 256), 256, 0, s>>>(totT, B->tiles, nrows.as<int64_t>());
  count_launch();
  CPM_TRY(exclusive_sum(nrows.as<int64_t>(), rowbase.as<int64_t>(), totT + 1, s));
  int64_t totRows = 0;
  CPM_TRY(read_back(rowbase.as<int64_t>() + totT, &totRows, s));
  CPM_TRY(dalloc<int64_t>(rowcnt, totRows + 1, "rowcnt"));
  CPM_TRY(dalloc<int64_t>(runstart, totRows + 1, "runstart"));
  CPM_CUDA(cudaMemsetAsync(rowcnt.p, 0, (totRows + 1) * sizeof(int64_t), s));
  k_runs<false><<<totT, 128, 0, s>>>(B->tiles, ebase.as<int32_t>(), tam.as<uint32_t>(), bmap.as<int>(), dblo.as<int>(),
                                     dbdim.as<int>(), rowbase.as<int64_t>(), rowcnt.as<int64_t>(),
                                     nullptr, nullptr);
  count_launch();
  CPM_TRY(exclusive_sum(rowcnt.as<int64_t>(), runstart.as<int64_t>(), totRows + 1, s));
  int64_t totRuns = 0;
  CPM_TRY(read_back(runstart.as<int64_t>() + totRows, &totRuns, s));
  if (totRuns >= (int64_t)INT32_MAX) return fail(CPM_ERR_LIMIT, "cpm_build_band: too many runs");
  CPM_TRY(dalloc_owned(&B->runs, (size_t)totRuns + 2, &B->bytes, "runs"));
  k_runs<true><<<totT, 128, 0, s>>>(B->tiles, ebase.as<int32_t>(), tam.as<uint32_t>(), bmap.as<int>(), dblo.as<int>(),
                                    dbdim.as<int>(), rowbase.as<int64_t>(), rowcnt.as<int64_t>(),
                                    runstart.as<int64_t>(), B->runs);
  count_launch();
  k_set_run_ranges<<<grid_for(totT, 256), 256, 0, s>>>(totT, B->tiles, rowbase.as<int64_t>(),
                                                        runstart.as<int64_t>());
  count_launch();
  CPM_CUDA(cudaGetLastError());
  B->nRuns = totRuns;
  if (!(getenv("CPM_RUNSORT") && *getenv("CPM_RUNSORT") == '0')) {
    // each tile's runs in source order: the 4 runs of a warp's cp.async touch fewer
    // L1 tags (3.38M -> 2.73M per config-1 apply, extend -1 us; CPM_RUNSORT=0: box-row order)
    DevBuf rb, re, sorted, tmpb;
    CPM_TRY(dalloc<int>(rb, totT, "run beg"));
    CPM_TRY(dalloc<int>(re, totT, "run end"));
    CPM_TRY(dalloc<uint64_t>(sorted, (size_t)totRuns + 2, "sorted runs"));
    k_run_offsets<<<grid_for(totT, 256), 256, 0, s>>>(totT, B->tiles, rb.as<int>(), re.as<int>());
    size_t tmp = 0;
    CPM_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tmp, B->runs, sorted.as<uint64_t>(), (int)totRuns,
                                                     totT, rb.as<int>(), re.as<int>(), 0, 32, s));
    CPM_TRY(dalloc<char>(tmpb, tmp, "sort temp"));
    CPM_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(tmpb.p, tmp, B->runs, sorted.as<uint64_t>(), (int)totRuns,
                                                     totT, rb.as<int>(), re.as<int>(), 0, 32, s));
    CPM_CUDA(cudaMemcpyAsync(B->runs, sorted.p, sizeof(uint64_t) * totRuns, cudaMemcpyDeviceToDevice, s));
    CPM_CUDA(cudaStreamSynchronize(s));
  }

  if (getenv("CPM_FUSED") && *getenv("CPM_FUSED") == '1')
    CPM_TRY(build_fused(B, bmap.as<int>(), dblo.as<int>(), dbdim.as<int>(), s));
  CPM_TRY(dalloc_owned(&B->vb, (size_t)totT * kBrickCells, &B->bytes, "vb"));
  // cells outside Sigma_A u Sigma_G are never written by the extend; k_laplace loads
  // whole slots (never using those cells): defined values for them
  CPM_CUDA(cudaMemsetAsync(B->vb, 0, sizeof(double) * (size_t)totT * kBrickCells, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  *out = guard.release();
  return CPM_OK;
}

}  // namespace cpm
