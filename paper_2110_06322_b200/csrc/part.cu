// part.cu — Morton-slab partition of the band across GPUs (north_star item 5).
//
// Rank r of R owns the band-order slab [lo, hi) = [floor(r nA / R), floor((r+1) nA / R))
// (reading R8).  Its local operator is a sub-band of the global band (every
// global rank builds the same band deterministically, so no geometry is
// communicated):
//   outputs  = owned active nodes (local index a - lo)
//   sources  = owned nodes + HALO nodes: the active nodes of other ranks that lie
//              in the stencil boxes of the tiles this rank evaluates (local index
//              n_owned + position in the sorted halo list)
//   tiles    = global tiles with an owned node or face-adjacent to one
// The stencil-box fill runs are the global band's runs re-indexed (split where
// they cross the owned range); the extend kernel reads owned sources from the
// Krylov vector and halo sources from a separate receive buffer, so no vector
// is ever copied into a [owned | halo] layout.
//
// Halo exchange (before every apply) and the Krylov inner products (after every
// reduction) go through NCCL, loaded at run time (dlopen libnccl.so.2: the
// library also loads on hosts without NCCL).
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "internal.cuh"
#include "krylov.cuh"
#include "part.cuh"
#include "ras.cuh"
#include "vecops.cuh"

namespace cpm {

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

int nccl_load() {
  if (g_nccl.ok) return CPM_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(CPM_ERR_NCCL, std::string("cannot dlopen libnccl.so.2: ") + dlerror());
#define LOADSYM(f)                                                            \
  g_nccl.f = (decltype(g_nccl.f))dlsym(h, "nccl" #f);                         \
  if (!g_nccl.f) return fail(CPM_ERR_NCCL, "libnccl.so.2 lacks nccl" #f);
  LOADSYM(GetUniqueId)
  LOADSYM(CommInitRank)
  LOADSYM(CommDestroy)
  LOADSYM(AllReduce)
  LOADSYM(Send)
  LOADSYM(Recv)
  LOADSYM(GroupStart)
  LOADSYM(GroupEnd)
  LOADSYM(GetErrorString)
#undef LOADSYM
  g_nccl.ok = true;
  return CPM_OK;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return CPM_OK;
  return fail(CPM_ERR_NCCL, std::string(what) + ": " + g_nccl.GetErrorString(r));
}
}  // namespace

// pinned host staging of a host-transport communicator, at least n doubles
static int host_stage(const cpm_comm* comm, size_t n) {
  cpm_comm* c = const_cast<cpm_comm*>(comm);
  if (c->cap >= n) return CPM_OK;
  if (c->stage) cudaFreeHost(c->stage);
  c->stage = nullptr;
  c->cap = 0;
  const size_t want = std::max<size_t>(n, 1024);
  CPM_CUDA(cudaMallocHost(&c->stage, want * sizeof(double)));
  c->cap = want;
  return CPM_OK;
}

int comm_allreduce_sum(const cpm_comm* comm, double* buf, size_t n, cudaStream_t s) {
  if (!comm || comm->nranks == 1 || n == 0) return CPM_OK;
  if (comm->host) {
    CPM_TRY(host_stage(comm, n));
    CPM_CUDA(cudaMemcpyAsync(comm->stage, buf, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CPM_CUDA(cudaStreamSynchronize(s));
    if (comm->ht.allreduce_sum(comm->ht.ctx, comm->stage, (int64_t)n) != 0)
      return fail(CPM_ERR_NCCL, "host transport: allreduce_sum callback failed");
    CPM_CUDA(cudaMemcpyAsync(buf, comm->stage, n * sizeof(double), cudaMemcpyHostToDevice, s));
    return CPM_OK;
  }
  return nccl_check(g_nccl.AllReduce(buf, buf, n, ncclDouble, ncclSum, (ncclComm_t)comm->nccl, s),
                    "ncclAllReduce");
}

namespace {

inline int g1(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

__global__ void k_owned_tiles(int nT, const TileHdr* tiles, int64_t lo, int64_t hi, int* has) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nT) has[t] = (tiles[t].a0 < hi && tiles[t].a1 > lo) ? 1 : 0;
}

__global__ void k_include(int nT, const TileHdr* tiles, const int* has, int* inc) {
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

// need[a] = 1 for every non-owned source of an included tile's fill runs;
// bnd[t] = 1 for an included tile with such a source (a BOUNDARY tile: its extend
// waits for the halo exchange), intr[t] = 1 for the other included tiles
__global__ void k_need(const TileHdr* tiles, const int* inc, const uint64_t* runs, int64_t lo,
                       int64_t hi, int* need, int* bnd, int* intr) {
  const int t = blockIdx.x;
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  if (inc[t]) {
    const TileHdr T = tiles[t];
    for (int r = T.r0 + threadIdx.x; r < T.r1; r += blockDim.x) {
      const uint64_t run = runs[r];
      const int64_t src = (uint32_t)run;
      const int len = (int)((run >> 48) & 0xff);
      for (int q = 0; q < len; ++q) {
        const int64_t a = src + q;
        if (a < lo || a >= hi) {
          need[a] = 1;
          any = 1;
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bnd[t] = inc[t] && any;
    intr[t] = inc[t] && !any;
  }
}

__global__ void k_flagged_index(int64_t n, const int* flag, const int* pos, int64_t* list) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n;
       a += (int64_t)gridDim.x * blockDim.x)
    if (flag[a]) list[pos[a]] = a;
}

// local source index of global active node a
__device__ __forceinline__ int64_t local_src(int64_t a, int64_t lo, int64_t hi, int64_t nOwned,
                                             const int* hpos) {
  return (a >= lo && a < hi) ? a - lo : nOwned + hpos[a];
}

// Re-index the included tiles' runs (split at lo and hi).  Thread per run.
template <bool WRITE>
__global__ void k_part_runs(int nT, const TileHdr* tiles, const int* inc, const uint64_t* runs,
                            int64_t lo, int64_t hi, int64_t nOwned, const int* hpos,
                            const int64_t* cntstart /*per global run*/, int64_t* cnt,
                            uint64_t* out) {
  const int t = blockIdx.x;
  if (!inc[t]) return;
  const TileHdr T = tiles[t];
  for (int r = T.r0 + threadIdx.x; r < T.r1; r += blockDim.x) {
    const uint64_t run = runs[r];
    const int64_t src = (uint32_t)run;
    const uint32_t dst = (uint32_t)(run >> 32) & 0xffffu;
    const int len = (int)((run >> 48) & 0xff);
    int n = 0;
    int q = 0;
    while (q < len) {
      const int64_t a = src + q;
      const bool own = a >= lo && a < hi;
      int q1 = q + 1;
      while (q1 < len && ((src + q1 >= lo && src + q1 < hi) == own)) ++q1;
      if (WRITE)
        out[cntstart[r] + n] =
            pack_run((uint32_t)local_src(a, lo, hi, nOwned, hpos), dst + q, (uint32_t)(q1 - q));
      ++n;
      q = q1;
    }
    if (!WRITE) cnt[r] = n;
  }
}

// sub-band tile order: the interior tiles first (Morton order), then the boundary
// tiles (Morton order), so the overlapped apply extends [0, nTint) while the halo
// exchange is in flight
__global__ void k_part_tiles(int nT, const TileHdr* tiles, const int* inc, const int* bnd,
                             const int* intpos, const int* bndpos, int nInt, int64_t lo, int64_t hi,
                             const int64_t* runstart, TileHdr* sub, int* tmap) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nT) return;
  if (!inc[t]) {
    tmap[t] = -1;
    return;
  }
  const int q = bnd[t] ? nInt + bndpos[t] : intpos[t];
  tmap[t] = q;
  TileHdr T = tiles[t];
  const int64_t a0 = std::max<int64_t>(T.a0, lo), a1 = std::min<int64_t>(T.a1, hi);
  T.a0 = (int32_t)(a0 < a1 ? a0 - lo : 0);
  T.a1 = (int32_t)(a0 < a1 ? a1 - lo : 0);
  T.r0 = (int32_t)runstart[tiles[t].r0];
  T.r1 = (int32_t)runstart[tiles[t].r1];
  T.pad[2] = 0;
  sub[q] = T;
}

__global__ void k_remap_nbrs(int n, TileHdr* sub, const int* tmap) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  for (int d = 0; d < 6; ++d) {
    const int g = sub[q].nbr[d];
    sub[q].nbr[d] = g >= 0 ? tmap[g] : -1;
  }
}

__global__ void k_gather_idx(int64_t n, const int64_t* idx, const double* x, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[idx[i]];
}

struct DB {
  void* p = nullptr;
  ~DB() {
    if (p) cudaFree(p);
  }
  int alloc(size_t bytes) {
    if (cudaMalloc(&p, std::max<size_t>(bytes, 16)) != cudaSuccess)
      return fail(CPM_ERR_NOMEM, "cpm_part_create: device allocation failed");
    return CPM_OK;
  }
  template <class T>
  T* as() const {
    return (T*)p;
  }
};

template <class T>
int scan(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  CPM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  DB tb;
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

}  // namespace


int part_create(const cpm_band* B, int rank, int R, cudaStream_t s, cpm_part** out) {
  if (!B || !out) return fail(CPM_ERR_ARG, "cpm_part_create: null argument");
  *out = nullptr;
  if (R < 1 || rank < 0 || rank >= R) return fail(CPM_ERR_ARG, "cpm_part_create: need 0 <= rank < nranks");
  if (!B->owns || B->nA < R) return fail(CPM_ERR_ARG, "cpm_part_create: needs a full band with n_active >= nranks");
  const int64_t nA = B->nA;
  const int nT = B->nT;
  auto P = std::make_unique<cpm_part>();
  P->band = B;
  P->rank = rank;
  P->nranks = R;
  P->lo = (int64_t)rank * nA / R;
  P->hi = (int64_t)(rank + 1) * nA / R;
  P->nOwned = P->hi - P->lo;
  for (int q = 0; q <= R; ++q) P->bounds.push_back((int64_t)q * nA / R);

  DB has, inc, incpos, need, hpos, tmap, bnd, intr, bndpos, intpos;
  CPM_TRY(has.alloc(sizeof(int) * (nT + 1)));
  CPM_TRY(inc.alloc(sizeof(int) * (nT + 1)));
  CPM_TRY(incpos.alloc(sizeof(int) * (nT + 1)));
  CPM_TRY(bnd.alloc(sizeof(int) * (nT + 1)));
  CPM_TRY(intr.alloc(sizeof(int) * (nT + 1)));
  CPM_TRY(bndpos.alloc(sizeof(int) * (nT + 1)));
  CPM_TRY(intpos.alloc(sizeof(int) * (nT + 1)));
  CPM_CUDA(cudaMemsetAsync(bnd.p, 0, sizeof(int) * (nT + 1), s));
  CPM_CUDA(cudaMemsetAsync(intr.p, 0, sizeof(int) * (nT + 1), s));
  CPM_TRY(need.alloc(sizeof(int) * (nA + 1)));
  CPM_TRY(hpos.alloc(sizeof(int) * (nA + 1)));
  CPM_TRY(tmap.alloc(sizeof(int) * nT));
  CPM_CUDA(cudaMemsetAsync(need.p, 0, sizeof(int) * (nA + 1), s));
  k_owned_tiles<<<(nT + 255) / 256, 256, 0, s>>>(nT, B->tiles, P->lo, P->hi, has.as<int>());
  count_launch();
  k_include<<<(nT + 256) / 256, 256, 0, s>>>(nT, B->tiles, has.as<int>(), inc.as<int>());
  count_launch();
  CPM_TRY(scan(inc.as<int>(), incpos.as<int>(), nT + 1, s));
  k_need<<<nT, 128, 0, s>>>(B->tiles, inc.as<int>(), B->runs, P->lo, P->hi, need.as<int>(), bnd.as<int>(),
                            intr.as<int>());
  count_launch();
  CPM_TRY(scan(bnd.as<int>(), bndpos.as<int>(), nT + 1, s));
  CPM_TRY(scan(intr.as<int>(), intpos.as<int>(), nT + 1, s));
  int nInt = 0;
  CPM_TRY(read1(intpos.as<int>() + nT, &nInt, s));
  CPM_TRY(scan(need.as<int>(), hpos.as<int>(), nA + 1, s));
  int nTs = 0, nH = 0;
  CPM_TRY(read1(incpos.as<int>() + nT, &nTs, s));
  CPM_TRY(read1(hpos.as<int>() + nA, &nH, s));
  P->nHalo = nH;
  CPM_CUDA(cudaMalloc(&P->halo, sizeof(int64_t) * std::max(nH, 1)));
  k_flagged_index<<<g1(nA), 256, 0, s>>>(nA, need.as<int>(), hpos.as<int>(), P->halo);
  count_launch();

  // runs: count, scan, write (per global run of included tiles)
  DB rcnt, rstart;
  CPM_TRY(rcnt.alloc(sizeof(int64_t) * (B->nRuns + 1)));
  CPM_TRY(rstart.alloc(sizeof(int64_t) * (B->nRuns + 1)));
  CPM_CUDA(cudaMemsetAsync(rcnt.p, 0, sizeof(int64_t) * (B->nRuns + 1), s));
  k_part_runs<false><<<nT, 128, 0, s>>>(nT, B->tiles, inc.as<int>(), B->runs, P->lo, P->hi, P->nOwned,
                                        hpos.as<int>(), nullptr, rcnt.as<int64_t>(), nullptr);
  count_launch();
  CPM_TRY(scan(rcnt.as<int64_t>(), rstart.as<int64_t>(), B->nRuns + 1, s));
  int64_t nR = 0;
  CPM_TRY(read1(rstart.as<int64_t>() + B->nRuns, &nR, s));
  cpm_band& L = P->lb;
  L.surf = B->surf;
  L.h = B->h;
  L.lam = B->lam;
  L.L = B->L;
  L.M = B->M;
  L.owns = false;
  L.nA = P->nOwned;
  L.nE = B->nE;
  L.nT = nTs;
  L.nTint = nInt;
  L.nRuns = nR;
  L.maxBox = B->maxBox;
  L.zeroFill = false;
  L.tx = B->tx;
  L.ty = B->ty;
  L.tz = B->tz;
  L.eoff = B->eoff;
  L.rnd = B->rnd;
  L.itemOrder = B->itemOrder;
  L.srcSplit = (uint32_t)P->nOwned;
  L.rank = rank;
  L.nranks = R;
  L.nOwned = P->nOwned;
  L.nHalo = nH;
  CPM_CUDA(cudaMalloc(&L.runs, sizeof(uint64_t) * std::max<int64_t>(nR, 1)));
  k_part_runs<true><<<nT, 128, 0, s>>>(nT, B->tiles, inc.as<int>(), B->runs, P->lo, P->hi, P->nOwned,
                                       hpos.as<int>(), rstart.as<int64_t>(), nullptr, L.runs);
  count_launch();
  CPM_CUDA(cudaMalloc(&L.tiles, sizeof(TileHdr) * std::max(nTs, 1)));
  k_part_tiles<<<(nT + 255) / 256, 256, 0, s>>>(nT, B->tiles, inc.as<int>(), bnd.as<int>(), intpos.as<int>(),
                                                bndpos.as<int>(), nInt, P->lo, P->hi, rstart.as<int64_t>(),
                                                L.tiles, tmap.as<int>());
  count_launch();
  k_remap_nbrs<<<(nTs + 255) / 256, 256, 0, s>>>(nTs, L.tiles, tmap.as<int>());
  count_launch();
  CPM_CUDA(cudaMalloc(&L.acell, sizeof(uint16_t) * std::max<int64_t>(P->nOwned, 1)));
  CPM_CUDA(cudaMemcpyAsync(L.acell, B->acell + P->lo, sizeof(uint16_t) * P->nOwned,
                           cudaMemcpyDeviceToDevice, s));
  CPM_CUDA(cudaMalloc(&L.vb, sizeof(double) * kBrickCells * (size_t)std::max(nTs, 1)));
  CPM_CUDA(cudaMemsetAsync(L.vb, 0, sizeof(double) * kBrickCells * (size_t)std::max(nTs, 1), s));
  CPM_CUDA(cudaMalloc(&P->hbuf, sizeof(double) * std::max(nH, 1)));
  CPM_CUDA(cudaGetLastError());

  // receive plan: halo is sorted by global index, hence grouped by owner rank
  std::vector<int64_t> hh(nH);
  if (nH > 0) CPM_CUDA(cudaMemcpyAsync(hh.data(), P->halo, sizeof(int64_t) * nH, cudaMemcpyDeviceToHost, s));
  CPM_CUDA(cudaStreamSynchronize(s));
  P->recvCount.assign(R, 0);
  P->recvOff.assign(R + 1, 0);
  for (int64_t a : hh) {
    const int q = (int)(std::upper_bound(P->bounds.begin(), P->bounds.end(), a) - P->bounds.begin()) - 1;
    P->recvCount[q]++;
  }
  for (int q = 0; q < R; ++q) P->recvOff[q + 1] = P->recvOff[q] + P->recvCount[q];
  if (P->recvCount[rank] != 0) return fail(CPM_ERR_GEOM, "cpm_part_create: halo contains owned nodes");
  P->ws = new Workspace();
  *out = P.release();
  return CPM_OK;
}

int part_set_send(cpm_part* P, const int64_t* send_global, const int64_t* counts) {
  if (!P || !counts) return fail(CPM_ERR_ARG, "cpm_part_set_send: null argument");
  const int R = P->nranks;
  P->sendCount.assign(counts, counts + R);
  P->sendOff.assign(R + 1, 0);
  for (int q = 0; q < R; ++q) {
    if (counts[q] < 0) return fail(CPM_ERR_ARG, "cpm_part_set_send: negative count");
    P->sendOff[q + 1] = P->sendOff[q] + counts[q];
  }
  const int64_t n = P->sendOff[R];
  std::vector<int64_t> loc(n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t a = send_global[i];
    if (a < P->lo || a >= P->hi) return fail(CPM_ERR_ARG, "cpm_part_set_send: requested node not owned");
    loc[i] = a - P->lo;
  }
  if (P->sendidx) cudaFree(P->sendidx);
  if (P->sendbuf) cudaFree(P->sendbuf);
  P->sendidx = nullptr;
  P->sendbuf = nullptr;
  CPM_CUDA(cudaMalloc(&P->sendidx, sizeof(int64_t) * std::max<int64_t>(n, 1)));
  CPM_CUDA(cudaMalloc(&P->sendbuf, sizeof(double) * std::max<int64_t>(n, 1)));
  if (n > 0) CPM_CUDA(cudaMemcpy(P->sendidx, loc.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice));
  P->nSend = n;
  return CPM_OK;
}

// Point-to-point exchange: gather x[sendidx] into sendbuf, then one NCCL group of
// send/recv per peer (peer q's slices at sendOff[q] / recvOff[q]) into recvbuf.
int halo_exchange(const cpm_comm* comm, int rank, int nranks, const double* x, int64_t nSend,
                  const int64_t* sendidx, double* sendbuf, const std::vector<int64_t>& sendCount,
                  const std::vector<int64_t>& sendOff, double* recvbuf,
                  const std::vector<int64_t>& recvCount, const std::vector<int64_t>& recvOff,
                  cudaStream_t s) {
  if (nranks == 1) return CPM_OK;
  if (!comm) return fail(CPM_ERR_ARG, "partitioned operation needs a communicator");
  if ((int)sendCount.size() != nranks) return fail(CPM_ERR_ARG, "halo exchange: send plan not set");
  if (nSend > 0) {
    k_gather_idx<<<g1(nSend), 256, 0, s>>>(nSend, sendidx, x, sendbuf);
    count_launch();
  }
  if (comm->host) {  // host-staged: [send | recv] in pinned staging, the caller's alltoallv
    const int64_t nRecv = recvOff[nranks];
    CPM_TRY(host_stage(comm, (size_t)(nSend + nRecv)));
    double* hs = comm->stage;
    double* hr = comm->stage + nSend;
    if (nSend > 0) CPM_CUDA(cudaMemcpyAsync(hs, sendbuf, nSend * sizeof(double), cudaMemcpyDeviceToHost, s));
    CPM_CUDA(cudaStreamSynchronize(s));
    if (comm->ht.alltoallv(comm->ht.ctx, hs, sendCount.data(), hr, recvCount.data()) != 0)
      return fail(CPM_ERR_NCCL, "host transport: alltoallv callback failed");
    if (nRecv > 0) CPM_CUDA(cudaMemcpyAsync(recvbuf, hr, nRecv * sizeof(double), cudaMemcpyHostToDevice, s));
    return CPM_OK;
  }
  CPM_TRY(nccl_check(g_nccl.GroupStart(), "ncclGroupStart"));
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) continue;
    if (sendCount[q] > 0)
      CPM_TRY(nccl_check(g_nccl.Send(sendbuf + sendOff[q], sendCount[q], ncclDouble, q,
                                     (ncclComm_t)comm->nccl, s), "ncclSend"));
    if (recvCount[q] > 0)
      CPM_TRY(nccl_check(g_nccl.Recv(recvbuf + recvOff[q], recvCount[q], ncclDouble, q,
                                     (ncclComm_t)comm->nccl, s), "ncclRecv"));
  }
  CPM_TRY(nccl_check(g_nccl.GroupEnd(), "ncclGroupEnd"));
  return CPM_OK;
}

// Halo exchange of the owned vector x into P->hbuf.
int part_exchange(const cpm_part* P, const cpm_comm* comm, const double* x, cudaStream_t s) {
  return halo_exchange(comm, P->rank, P->nranks, x, P->nSend, P->sendidx, P->sendbuf, P->sendCount,
                       P->sendOff, P->hbuf, P->recvCount, P->recvOff, s);
}

// y = A x on the owned slice.  With several ranks the halo exchange (gather + NCCL
// send/recv, or the host transport) runs on a side stream while the interior tiles
// (no halo source: [0, nTint) of the sub-band) are extended on s; the boundary tiles'
// extend waits for the exchange, then the laplace of all tiles.  CPM_HALO_OVERLAP=0:
// exchange, then the whole apply (A/B).
int part_apply(const cpm_part* P, const cpm_comm* comm, double c, const double* x, double* y,
               const double* scale, const int* skip, cudaStream_t s) {
  static const bool overlap = [] {
    const char* v = getenv("CPM_HALO_OVERLAP");
    return !v || *v != '0';
  }();
  const cpm_band* L = &P->lb;
  if (P->nranks == 1 || !overlap) {
    CPM_TRY(part_exchange(P, comm, x, s));  // collective: always performed
    return apply_device_split(L, c, x, P->hbuf, y, scale, 0, s, skip);
  }
  cpm_part* mp = const_cast<cpm_part*>(P);
  if (!mp->xs || !mp->xev[0] || !mp->xev[1]) {  // (a failed earlier attempt leaves nulls)
    if (!mp->xs) CPM_CUDA(cudaStreamCreateWithFlags(&mp->xs, cudaStreamNonBlocking));
    if (!mp->xev[0]) CPM_CUDA(cudaEventCreateWithFlags(&mp->xev[0], cudaEventDisableTiming));
    if (!mp->xev[1]) CPM_CUDA(cudaEventCreateWithFlags(&mp->xev[1], cudaEventDisableTiming));
  }
  CPM_CUDA(cudaEventRecord(mp->xev[0], s));  // x produced; the previous apply read hbuf
  CPM_CUDA(cudaStreamWaitEvent(mp->xs, mp->xev[0], 0));
  if (L->nT > 0) CPM_TRY(extend_tiles(L, x, P->hbuf, s, skip, 0, L->nTint));
  CPM_TRY(part_exchange(P, comm, x, mp->xs));
  CPM_CUDA(cudaEventRecord(mp->xev[1], mp->xs));
  CPM_CUDA(cudaStreamWaitEvent(s, mp->xev[1], 0));
  if (L->nT == 0) return CPM_OK;
  CPM_TRY(extend_tiles(L, x, P->hbuf, s, skip, L->nTint, L->nT));
  return laplace_tiles(L, c, x, y, scale, 0, s, skip);
}

}  // namespace cpm

cpm_comm::~cpm_comm() {
  if (stage) cudaFreeHost(stage);
}

cpm_part::~cpm_part() {
  void* ps[] = {lb.tiles, lb.runs, lb.vb, lb.acell, halo, hbuf, sendidx, sendbuf, rdstage};
  for (void* p : ps)
    if (p) cudaFree(p);
  if (xs) cudaStreamDestroy(xs);
  for (cudaEvent_t e : xev)
    if (e) cudaEventDestroy(e);
  lb.tiles = nullptr;
  delete ws;
}

using namespace cpm;

extern "C" {

int cpm_comm_unique_id(void* id_out) {
  if (!id_out) return fail(CPM_ERR_ARG, "cpm_comm_unique_id: null");
  CPM_TRY(nccl_load());
  ncclUniqueId id;
  CPM_TRY(nccl_check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId"));
  memcpy(id_out, &id, sizeof(id));
  return CPM_OK;
}

int cpm_comm_init(const void* id, int rank, int nranks, cpm_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(CPM_ERR_ARG, "cpm_comm_init: bad arguments");
  *out = nullptr;
  CPM_TRY(nccl_load());
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c;
  CPM_TRY(nccl_check(g_nccl.CommInitRank(&c, nranks, uid, rank), "ncclCommInitRank"));
  cpm_comm* cm = new cpm_comm();
  cm->nccl = c;
  cm->rank = rank;
  cm->nranks = nranks;
  *out = cm;
  return CPM_OK;
}

int cpm_comm_init_host(const cpm_host_transport* tr, int rank, int nranks, cpm_comm** out) {
  if (!tr || !out || !tr->allreduce_sum || !tr->alltoallv || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(CPM_ERR_ARG, "cpm_comm_init_host: bad arguments");
  cpm_comm* cm = new cpm_comm();
  cm->host = true;
  cm->ht = *tr;
  cm->rank = rank;
  cm->nranks = nranks;
  *out = cm;
  return CPM_OK;
}

void cpm_comm_free(cpm_comm* c) {
  if (!c) return;
  if (c->nccl && g_nccl.ok) g_nccl.CommDestroy((ncclComm_t)c->nccl);
  delete c;
}

int cpm_part_create(const cpm_band* band, int rank, int nranks, void* stream, cpm_part** out) {
  return part_create(band, rank, nranks, (cudaStream_t)stream, out);
}

int cpm_part_get_info(const cpm_part* p, cpm_part_info* info) {
  if (!p || !info) return fail(CPM_ERR_ARG, "cpm_part_get_info: null");
  memset(info, 0, sizeof(*info));
  info->rank = p->rank;
  info->nranks = p->nranks;
  info->lo = p->lo;
  info->hi = p->hi;
  info->n_owned = p->nOwned;
  info->n_halo = p->nHalo;
  info->n_tiles = p->lb.nT;
  info->n_send = p->nSend;
  info->n_interior_tiles = p->lb.nTint;
  return CPM_OK;
}

int cpm_part_halo_nodes(const cpm_part* p, int64_t* host_out) {
  if (!p || (!host_out && p->nHalo > 0)) return fail(CPM_ERR_ARG, "cpm_part_halo_nodes: null");
  if (p->nHalo > 0)
    CPM_CUDA(cudaMemcpy(host_out, p->halo, sizeof(int64_t) * p->nHalo, cudaMemcpyDeviceToHost));
  return CPM_OK;
}

int cpm_part_set_send(cpm_part* p, const int64_t* send_global, const int64_t* counts) {
  return part_set_send(p, send_global, counts);
}

int cpm_part_apply_local(const cpm_part* p, double c, const double* u_owned, const double* u_halo,
                         double* y_owned, void* stream) {
  if (!p || !u_owned || !y_owned || (p->nHalo > 0 && !u_halo))
    return fail(CPM_ERR_ARG, "cpm_part_apply_local: null argument");
  if (!is_device_ptr(u_owned) || !is_device_ptr(y_owned) || (p->nHalo > 0 && !is_device_ptr(u_halo)))
    return fail(CPM_ERR_ARG, "cpm_part_apply_local: vectors must be device memory");
  return apply_device_split(&p->lb, c, u_owned, u_halo, y_owned, nullptr, 0, (cudaStream_t)stream);
}

int cpm_part_apply(const cpm_part* p, const cpm_comm* comm, double c, const double* u_owned,
                   double* y_owned, void* stream) {
  if (!p || !u_owned || !y_owned) return fail(CPM_ERR_ARG, "cpm_part_apply: null argument");
  if (!is_device_ptr(u_owned) || !is_device_ptr(y_owned))
    return fail(CPM_ERR_ARG, "cpm_part_apply: vectors must be device memory");
  if (p->nranks > 1 && !comm) return fail(CPM_ERR_ARG, "cpm_part_apply: needs a communicator");
  return part_apply(p, comm, c, u_owned, y_owned, nullptr, nullptr, (cudaStream_t)stream);
}

static int part_solve(const cpm_part* p, const cpm_comm* comm, double c, const double* f_owned,
                      double* u_owned, double rtol, int restart, int maxit, const cpm_ras* ras,
                      cpm_solve_stats* stats, void* stream);

int cpm_part_solve(const cpm_part* p, const cpm_comm* comm, double c, const double* f_owned,
                   double* u_owned, double rtol, int restart, int maxit, const cpm_ras* ras,
                   cpm_solve_stats* stats, void* stream) {
  if (!p || !f_owned || !u_owned) return fail(CPM_ERR_ARG, "cpm_part_solve: null argument");
  if (!is_device_ptr(f_owned) || !is_device_ptr(u_owned))
    return fail(CPM_ERR_ARG, "cpm_part_solve: vectors must be device memory");
  if (p->nranks > 1 && !comm) return fail(CPM_ERR_ARG, "cpm_part_solve: needs a communicator");
  return part_solve(p, comm, c, f_owned, u_owned, rtol, restart, maxit, ras, stats, stream);
}

int cpm_part_rd_step(const cpm_part* p, const cpm_comm* comm, const cpm_rd_params* prm, double* u_owned,
                     double* v_owned, cpm_solve_stats* su, cpm_solve_stats* sv, void* stream) {
  if (!p || !prm || !u_owned || !v_owned) return fail(CPM_ERR_ARG, "cpm_part_rd_step: null argument");
  if (u_owned == v_owned) return fail(CPM_ERR_ARG, "cpm_part_rd_step: u and v must not alias");
  if (!(prm->dt > 0.0) || !(prm->mu1 > 0.0) || !(prm->mu2 > 0.0))
    return fail(CPM_ERR_ARG, "cpm_part_rd_step: dt, mu1, mu2 must be > 0");
  if (!is_device_ptr(u_owned) || !is_device_ptr(v_owned))
    return fail(CPM_ERR_ARG, "cpm_part_rd_step: vectors must be device memory");
  if (p->nranks > 1 && !comm) return fail(CPM_ERR_ARG, "cpm_part_rd_step: needs a communicator");
  cudaStream_t s = (cudaStream_t)stream;
  cpm_part* mp = const_cast<cpm_part*>(p);
  if (!mp->rdstage) CPM_CUDA(cudaMalloc(&mp->rdstage, sizeof(double) * 2 * std::max<int64_t>(p->nOwned, 1)));
  double* ru = mp->rdstage;
  double* rv = mp->rdstage + std::max<int64_t>(p->nOwned, 1);
  const double c1 = 1.0 / (prm->dt * prm->mu1), c2 = 1.0 / (prm->dt * prm->mu2);
  // the reaction terms on the owned slice (pointwise: no exchange), then two shifted
  // partitioned solves warm-started from the old state (reading R14)
  CPM_TRY(rd_rhs_device(p->nOwned, u_owned, v_owned, prm, c1, c2, ru, rv, s));
  cpm_solve_stats l1, l2;
  CPM_TRY(part_solve(p, comm, c1, ru, u_owned, prm->rtol, prm->restart, prm->maxit, nullptr, su ? su : &l1, s));
  CPM_TRY(part_solve(p, comm, c2, rv, v_owned, prm->rtol, prm->restart, prm->maxit, nullptr, sv ? sv : &l2, s));
  return CPM_OK;
}

static int part_solve(const cpm_part* p, const cpm_comm* comm, double c, const double* f_owned,
                      double* u_owned, double rtol, int restart, int maxit, const cpm_ras* ras,
                      cpm_solve_stats* stats, void* stream) {
  PrecOp M;
  if (ras) {
    cpm_ras_info ri;
    CPM_TRY(cpm_ras_get_info(ras, &ri));
    if (ras->band != p->band || ri.rank != p->rank || ri.nranks != p->nranks)
      return fail(CPM_ERR_ARG, "cpm_part_solve: preconditioner built for another partition");
    M.apply = [ras, comm](const double* r, double* z, cudaStream_t st) {
      CPM_TRY(ras_exchange(ras, comm, r, st));
      return ras_apply_device(ras, r, z, st);
    };
  }
  LinOp A;
  A.apply = [p, comm, c](const double* x, double* y, const double* scale, const int* skip,
                         cudaStream_t st) {
    return part_apply(p, comm, c, x, y, scale, skip, st);  // the exchange is collective: always performed
  };
  A.allreduce = [comm](double* buf, size_t n, cudaStream_t st) { return comm_allreduce_sum(comm, buf, n, st); };
  cpm_solve_stats local;
  return gmres_device(A, ras ? &M : nullptr, f_owned, u_owned, p->nOwned, rtol, restart, maxit, *p->ws,
                      stats ? stats : &local, (cudaStream_t)stream);
}

void cpm_part_free(cpm_part* p) { delete p; }

}  // extern "C"
